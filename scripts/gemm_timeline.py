"""Per-CTA phase timeline of one GEMM launch (dbg bit 8 timestamps)."""
import ctypes as C, json, sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X
kind = int(sys.argv[1]); B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
L, d = 12, 768
cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique.never(), max_batch=B,
                     pool_blocks=B * L * 40, eos_token=-1)
e = X.Engine(cfg)
e.set_option("dbg", 8)
e.session_begin(np.arange(B) + 1, 511, 640, 1)
lib = X.lib(); lib.el_debug_timestamps.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
for rep in range(2):
    ms = e.time_kernel(kind, 1, 1)
    ts = np.zeros(65536, np.uint64)
    lib.el_debug_timestamps(e._h, ts.ctypes.data_as(C.c_void_p), 65536)
info = e.plan_info()
n = {1: info["qkv_splits"] * 18, 2: info["wo_splits"] * 6, 3: info["up_splits"] * 24, 4: info["down_splits"] * 6, 5: 251}[kind]
t = ts[: n * 8].reshape(n, 8).astype(np.int64)
t0 = t[:, 0].min()
names = ["start", "tmem+bar", "prologue", "accf", "csync1", "reduce", "done", "dealloc"]
for i, nm in enumerate(names):
    col = t[:, i]; col = col[col > 0] - t0
    if len(col): print(f"{nm:10s} min {col.min()/1e3:7.2f}us  med {np.median(col)/1e3:7.2f}us  max {col.max()/1e3:7.2f}us")
print("kernel ms (event, incl. launch):", ms)
