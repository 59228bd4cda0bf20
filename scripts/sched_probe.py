"""Layer-level scheduling smoke (debug helper): a few turns at small dims, printing each turn."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402
L, d, V, B = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (6, 256, 1024, 24)))
turns = int(sys.argv[5]) if len(sys.argv) > 5 else 6
cfg = X.EngineConfig(model=X.ModelConfig(L, d, V, 0), technique=X.ExitTechnique("state"),
                     schedule=X.ThresholdSchedule(0.97, 0.998, 0.0), max_batch=B, pool_blocks=B * L * 16, eos_token=-1)
e = X.Engine(cfg)
e.session_begin(np.arange(B) + 1, 40, 105, 1, np.arange(B))
e.sched_begin("greedy")
for t in range(turns):
    e.sched_run(1)
    la, ro = e.sched_turns()
    print("turn", t, "layer", la[-1], "rows", ro[-1], "tokens", sum(len(e.sched_tokens(b)[0]) for b in range(B)), flush=True)
