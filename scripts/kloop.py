"""k-block timeline of CTA 0 of one GEMM launch (dbg bit 16)."""
import ctypes as C, sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X
kind, cap = int(sys.argv[1]), int(sys.argv[2])
L, d, B = 12, 768, 64
cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique.never(), max_batch=B,
                     pool_blocks=B * L * 40, eos_token=-1)
e = X.Engine(cfg); e.set_option("splits_cap", cap); e.set_option("dbg", 24)
e.session_begin(np.arange(B) + 1, 511, 640, 1)
lib = X.lib(); lib.el_debug_timestamps.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
for _ in range(2):
    e.time_kernel(kind, 1, 1)
ts = np.zeros(65536, np.uint64); lib.el_debug_timestamps(e._h, ts.ctypes.data_as(C.c_void_p), 65536)
t0 = int(ts[0])  # CTA 0 start
full = ts[4096:4096 + 64].astype(np.int64); emp = ts[4160:4160 + 64].astype(np.int64)
print("cta0 phases (us):", [(i, round((int(ts[i]) - t0) / 1e3, 2)) for i in range(8) if ts[i]])
print("full-ready (us): ", [round((x - t0) / 1e3, 2) for x in full if x > 0])
print("empty-ready (us):", [round((x - t0) / 1e3, 2) for x in emp if x > 0])
