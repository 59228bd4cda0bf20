"""Option sweep of the persistent decode-iteration kernel: us/iteration (full depth, technique never)
and the early-exit bench technique.  python scripts/mega_sweep.py c2 '[{"mega_att_stages": 2}, ...]'"""
import json
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402

DIMS = {"c1": (6, 512, 8), "c2": (12, 768, 64), "c3": (24, 1024, 128), "c5": (24, 1024, 256)}
cfgname = sys.argv[1]
variants = json.loads(sys.argv[2])
techs = sys.argv[3].split(",") if len(sys.argv) > 3 else ["never"]
L, d, B = DIMS[cfgname]
for tech in techs:
    cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique(tech, 4),
                         schedule=X.ThresholdSchedule(0.981, 0.997, 0.0), max_batch=B, pool_blocks=B * L * 42,
                         eos_token=-1)
    e = X.Engine(cfg, mega=True)
    for v in variants:
        for k, x in v.items():
            e.set_option(k, x)
        e.session_begin(np.arange(B) + 1, 511, 660, 1)
        e.decode_run(3)
        ms = e.time_decode(20) / 20
        print(f"{cfgname} {tech:8s} {json.dumps(v):50s} {ms * 1e3:8.1f} us/iter", flush=True)
        e.session_end()
    e.close()
