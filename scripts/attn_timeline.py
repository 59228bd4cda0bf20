"""Block-level timeline of the first 4 attention CTAs (dbg bit 32)."""
import ctypes as C, json, sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X
opts = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {}
L, d, B = 12, 768, 64
cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique.never(), max_batch=B,
                     pool_blocks=B * L * 40, eos_token=-1)
e = X.Engine(cfg)
for kk, v in opts.items(): e.set_option(kk, v)
e.set_option("dbg", 32 | opts.get("dbg", 0))
e.session_begin(np.arange(B) + 1, 511, 640, 1)
lib = X.lib(); lib.el_debug_timestamps.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
for _ in range(3): ms = e.time_kernel(0, 1, 1)
ts = np.zeros(65536, np.uint64); lib.el_debug_timestamps(e._h, ts.ctypes.data_as(C.c_void_p), 65536)
starts = ts[8192 + 512: 8192 + 516].astype(np.int64); t0 = starts.min()
for c in range(2):
    full = ts[8192 + c * 128: 8192 + c * 128 + 60].astype(np.int64)
    iss = ts[8192 + c * 128 + 64: 8192 + c * 128 + 124].astype(np.int64)
    print(f"cta{c} start {(starts[c]-t0)/1e3:.2f}us")
    print("  issue:", [round((x - t0) / 1e3, 2) for x in iss if x > 0][:30])
    print("  full :", [round((x - t0) / 1e3, 2) for x in full if x > 0][:30])
print("event ms", ms, e.plan_info())
g = 148
t = ts[24576:24576 + 4 * g].reshape(g, 4).astype(np.int64)
t0 = t[:, 0].min()
for i, nm in enumerate(["start", "first_full", "last_full(term)", "end"]):
    col = (t[:, i] - t0) / 1e3
    print(f"{nm:16s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f}  argmax {col.argmax()}")
