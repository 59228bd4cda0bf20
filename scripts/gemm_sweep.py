"""GEMM kernel time per kind vs split cap (events, standalone) + timeline medians."""
import ctypes as C, json, sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X
L, d, B = 12, 768, int(sys.argv[1]) if len(sys.argv) > 1 else 64
for cap in [1, 2, 4, 8]:
    cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique.never(), max_batch=B,
                         pool_blocks=B * L * 40, eos_token=-1)
    e = X.Engine(cfg)
    e.set_option("splits_cap", cap)
    e.session_begin(np.arange(B) + 1, 511, 640, 1)
    kt = {name: round(e.time_kernel(kind, 1, 20) * 1e3, 1) for kind, name in [(1, "qkv"), (2, "wo"), (3, "up"), (4, "down")]}
    print(json.dumps(dict(B=B, splits_cap=cap, kernels_us=kt, plan=e.plan_info())), flush=True)
    e.close()
