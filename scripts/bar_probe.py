"""Grid-barrier cost inside the persistent kernel (dbg 256: 32 empty barriers at kernel start)."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402

L, d, B = 2, 768, 64
cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique("never"), max_batch=B,
                     pool_blocks=B * L * 40, eos_token=-1)
e = X.Engine(cfg)
e.session_begin(np.arange(B) + 1, 511, 640, 1)
lib = X.lib()
lib.el_debug_timestamps.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
e.decode_run(2)
for name, dbg in (("A full fences", 0), ("A no proxy fence", 512), ("A no threadfence", 1024), ("B backoff", 2048),
                  ("C flags", 4096), ("C flags no proxy", 4096 | 512), ("D master", 8192), ("D no proxy", 8192 | 512),
                  ("E relaxed poll", 16384), ("E no proxy", 16384 | 512), ("F flags relaxed", 32768),
                  ("F no proxy", 32768 | 512)):
    e.set_option("dbg", 128 | 256 | dbg)
    e.decode_run(1)
    e.sync()
    ts = np.zeros(65536, np.uint64)
    lib.el_debug_timestamps(e._h, ts.ctypes.data_as(C.c_void_p), 65536)
    t = ts[20480:20480 + 33].astype(np.float64)
    dt = np.diff(t) / 1e3
    ms = e.time_decode(5) / 5
    print(f"{name:18s} iteration {ms * 1e3:8.1f} us  barrier mean {dt.mean():.3f} us  min {dt.min():.3f}  max {dt.max():.3f}")
