"""Decode-iteration time (product build, persistent kernel) under option sets, same session:
    python scripts/opt_time.py c2 state '{}' '{"mega_down_splits":12}' ..."""
import json
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402

DIMS = {"c2": (12, 768, 64, 0.981, 0.997), "c3": (24, 1024, 128, 0.41, 0.997), "c5": (24, 1024, 256, 0.41, 0.997)}
name, tech = sys.argv[1], sys.argv[2]
L, d, B, lam, gam = DIMS[name]
for rep in range(2):
    for o in sys.argv[3:]:
        cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique(tech, 4),
                             schedule=X.ThresholdSchedule(lam, gam, 0.0), max_batch=B, pool_blocks=B * L * 42,
                             eos_token=-1)
        e = X.Engine(cfg, mega=True)
        for k, v in json.loads(o).items():
            e.set_option(k, v)
        e.session_begin(np.arange(B) + 1, 511, 660, 1)
        e.decode_run(5)
        e.sync()
        us = e.time_decode(40) / 40 * 1e3
        print(f"{name} {tech} {o:40s} {us:8.1f} us/iteration")
        e.close()
