"""Layer-level scheduling turn cost at c5 dims (classifier, bench thresholds): wall time per turn
(host round trip included) and, under ncu, the turn kernel's own duration.
    python scripts/ll_probe.py [turns]"""
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402

turns = int(sys.argv[1]) if len(sys.argv) > 1 else 40
B, L, d, prefix = 256, 24, 1024, 511
cap = prefix + 1 + 2 * L + turns + 2
cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique("classifier"),
                     schedule=X.ThresholdSchedule(0.41, 0.997, 0.0), max_batch=B, pool_blocks=B * L * (-(-cap // 16)),
                     eos_token=-1)
e = X.Engine(cfg)
e.session_begin(np.arange(B) + 1, prefix, cap, 1, np.arange(B))
e.sched_begin("greedy")
e.sched_run(2 * L)
ms = e.sched_run(turns)
tl, tr = e.sched_turns()
print(f"{ms / turns * 1e3:.1f} us per turn (wall, host round trip incl.), mean rows per turn "
      f"{tr[2 * L:].mean():.1f}, layers {np.bincount(tl[2 * L:], minlength=L + 1)[1:].tolist()}")
