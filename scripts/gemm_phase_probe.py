"""Per-phase strategy (one kernel per GEMM phase, host-driven layer loop) at a BASELINE config, for
ncu -k regex:gemm_kernel: each projection GEMM (QKV, W_o, up, down) and the LM head is its own
launch, so ncu reports tensor-pipe and DRAM utilisation per GEMM.
    python scripts/gemm_phase_probe.py [c2|c3|c5] [n_iters]"""
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402

DIMS = {"c2": (12, 768, 64), "c3": (24, 1024, 128), "c5": (24, 1024, 256)}
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
L, d, B = DIMS[name]
cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique("always_at", 2), max_batch=B,
                     pool_blocks=B * L * 42, eos_token=-1)
e = X.Engine(cfg, graph=False, mega=False)
e.session_begin(np.arange(B) + 1, 511, 660, 1)
e.decode_run(n)
e.sync()
print("ok", e.records(0, n)["output_layer"].tolist())
