"""f1 measurement: Engine::run prefill throughput (prompt positions / s) at C2 dims, batched causal
prefill on the persistent kernel vs the per-position per-phase path.  Each request generates 1 token,
so the run is dominated by the prefill of its 511 prompt positions (engine.cpp:166-181)."""
import sys
import time

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402

L, d, V = 12, 768, 32128
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
P = int(sys.argv[2]) if len(sys.argv) > 2 else 512
rng = np.random.default_rng(1)
reqs = [X.Request(0.0, [int(x) for x in rng.integers(1, V, P)], 1) for _ in range(B)]
for mega in (True, False):
    cfg = X.EngineConfig(model=X.ModelConfig(L, d, V, 0), technique=X.ExitTechnique("never"), max_batch=B,
                         pool_blocks=B * L * (P // 16 + 2), eos_token=-1)
    e = X.Engine(cfg, mega=mega)
    e.run(X.Workload(reqs[:2]))  # warm-up (plans, graphs)
    t0 = time.perf_counter()
    t = e.run(X.Workload(reqs))
    dt = time.perf_counter() - t0
    print(f"{'persistent batched' if mega else 'per-position per-phase'} prefill: {B} x {P - 1} positions in "
          f"{dt * 1e3:.1f} ms -> {B * (P - 1) / dt:,.0f} positions/s", flush=True)
    e.close()
