"""Run a few persistent-kernel decode iterations on a bench-shaped session (for ncu -k iter_kernel -s 2 -c 1).
    python scripts/iter_only.py [c1|c2|c3|c4m|c5] [technique] [n_iters]"""
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402

DIMS = {"c1": (6, 512, 8, 1e-7, 1.0), "c2": (12, 768, 64, 0.981, 0.997), "c3": (24, 1024, 128, 0.41, 0.997),
        "c5": (24, 1024, 256, 0.41, 0.997), "c4m": (24, 1024, 128, 7e-8, 1.0), "c2t5": (12, 768, 64, 0.981, 0.997), "c5t5": (24, 1024, 256, 0.41, 0.997)}
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
tech = sys.argv[2] if len(sys.argv) > 2 else "never"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 3
L, d, B, lam, gam = DIMS[name]
enc = 512 if name.endswith("t5") else 0
cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0, encoder_len=enc), technique=X.ExitTechnique(tech),
                     schedule=X.ThresholdSchedule(lam, gam, 0.0), max_batch=B, pool_blocks=B * L * 42, eos_token=-1)
e = X.Engine(cfg, mega=True)
e.session_begin(np.arange(B) + 1, 63 if enc else 511, 660, 1)
e.decode_run(n)
e.sync()
print("ok", e.records(0, n)["output_layer"].tolist())
