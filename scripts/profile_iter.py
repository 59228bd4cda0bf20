"""Set up a bench-shaped decode session and run a few iterations (for ncu)."""
import argparse, sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X

ap = argparse.ArgumentParser()
ap.add_argument("--L", type=int, default=12); ap.add_argument("--d", type=int, default=768)
ap.add_argument("--B", type=int, default=64); ap.add_argument("--tech", default="state")
ap.add_argument("--lam", type=float, default=0.972); ap.add_argument("--gamma", type=float, default=0.998)
ap.add_argument("--iters", type=int, default=2); ap.add_argument("--warm", type=int, default=2)
ap.add_argument("--graph", type=int, default=1); ap.add_argument("--exit_layer", type=int, default=1)
a = ap.parse_args()
V, P = 32128, 512
cfg = X.EngineConfig(model=X.ModelConfig(a.L, a.d, V, 0), technique=X.ExitTechnique(a.tech, a.exit_layer),
                     schedule=X.ThresholdSchedule(a.lam, a.gamma, 0.0), max_batch=a.B,
                     pool_blocks=a.B * a.L * 40, eos_token=-1)
e = X.Engine(cfg, graph=bool(a.graph))
rng = np.random.default_rng(1)
e.session_begin(rng.integers(1, V, a.B), P - 1, 640, 1)
print("plan", e.plan_info())
for _ in range(a.warm):
    r = e.decode_iteration()
e.sync()
t = time.time()
e.decode_run(a.iters); e.sync()
rec = e.records(a.warm, a.iters)
print("out layers", rec["output_layer"].tolist(), "wall ms/iter", (time.time() - t) * 1e3 / a.iters)
