"""Launch one kernel kind a few times on a bench-shaped session (for ncu -s 1 -c 1)."""
import json, sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X
kind = int(sys.argv[1]); L = int(sys.argv[2]) if len(sys.argv) > 2 else 12
d = int(sys.argv[3]) if len(sys.argv) > 3 else 768; B = int(sys.argv[4]) if len(sys.argv) > 4 else 64
opts = json.loads(sys.argv[5]) if len(sys.argv) > 5 else {}
cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique.never(), max_batch=B,
                     pool_blocks=B * L * 40, eos_token=-1)
e = X.Engine(cfg)
for k, v in opts.items():
    e.set_option(k, v)
e.session_begin(np.arange(B) + 1, 511, 640, 1)
print(kind, opts, e.time_kernel(kind, 1, 3) * 1e3, "us", e.plan_info())
