"""Attention pipeline of layer 1 inside the persistent kernel (dbg 32|128): per block issue time
(producer) vs consume time (consumer warps) for CTAs 0-3, relative to the CTA's phase start."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402

DIMS = {"c2": (12, 768, 64), "c5": (24, 1024, 256)}
L, d, B = DIMS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique("always_at", 1), max_batch=B,
                     pool_blocks=B * L * 42, eos_token=-1)
e = X.Engine(cfg, mega=True)
e.session_begin(np.arange(B) + 1, 511, 660, 1)
lib = X.lib()
lib.el_debug_timestamps.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
e.decode_run(2)
e.sync()
e.set_option("dbg", 32 | 128)
e.decode_run(1)
e.sync()
ts = np.zeros(65536 + 256 * 1024, np.uint64)
lib.el_debug_timestamps(e._h, ts.ctypes.data_as(C.c_void_p), ts.size)
A = ts[40000:40000 + 512].reshape(256, 2).astype(np.float64)  # layer 1 attention phase start/end per CTA
for cta in range(4):
    t0 = A[cta, 0]
    iss = ts[8192 + 1024 + cta * 128: 8192 + 1024 + cta * 128 + 60].astype(np.float64)
    con = ts[8192 + cta * 128: 8192 + cta * 128 + 60].astype(np.float64)
    n = int(np.argmax(iss == 0)) if (iss == 0).any() else 60
    print(f"CTA {cta}: phase {(A[cta, 1] - t0) / 1e3:.2f} us, {n} stages")
    print("  issue  :", " ".join(f"{(x - t0) / 1e3:5.1f}" for x in iss[:n]))
    print("  consume:", " ".join(f"{(x - t0) / 1e3:5.1f}" for x in con[:n + 1]))
    don = ts[8192 + 2048 + cta * 128: 8192 + 2048 + cta * 128 + 60].astype(np.float64)
    print("  done   :", " ".join(f"{(x - t0) / 1e3:5.1f}" for x in don[:n]))
    print("  proc us:", " ".join(f"{(x - y) / 1e3:5.2f}" for x, y in zip(don[:n], con[:n])))
