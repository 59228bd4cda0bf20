"""Block-level timeline of attention CTAs 0..3 in the standalone attn_kernel (EL_DEBUG build, dbg 32):
per ring slot the producer's issue time, the consumers' full-barrier pass and the block-processed
time.  Usage: python scripts/attn_tl2.py [B] [d] [ctas] [stages]"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
d = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
ctas = int(sys.argv[3]) if len(sys.argv) > 3 else 148
S = int(sys.argv[4]) if len(sys.argv) > 4 else 2
L = 4
cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique("never"), max_batch=B,
                     pool_blocks=B * L * 40, eos_token=-1)
e = X.Engine(cfg, mega=False)
e.session_begin(np.arange(B) + 1, 511, 640, 1)
e.set_option("attn_stages", S)
e.set_option("attn_grid", ctas)
e.set_option("dbg", 32)
lib = X.lib()
lib.el_debug_timestamps.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
for _ in range(3):
    ms = e.time_kernel(0x100, 1, 1)
ts = np.zeros(65536, np.uint64)
lib.el_debug_timestamps(e._h, ts.ctypes.data_as(C.c_void_p), 65536)
print(f"B {B} d {d} ctas {ctas} stages {S}: launch {ms * 1e3:.1f} us")
for c in range(2):
    iss = ts[8192 + 1024 + c * 128: 8192 + 1024 + c * 128 + 60].astype(np.int64)
    full = ts[8192 + c * 128: 8192 + c * 128 + 60].astype(np.int64)
    done = ts[8192 + 2048 + c * 128: 8192 + 2048 + c * 128 + 60].astype(np.int64)
    t0 = iss[iss > 0].min()
    n = int((iss > 0).sum())
    print(f"cta {c}: {n} blocks")
    for i in range(min(n, 40)):
        f = (full[i] - t0) / 1e3 if full[i] else -1
        dn = (done[i] - t0) / 1e3 if done[i] else -1
        print(f"  blk {i:2d} issue {(iss[i] - t0) / 1e3:7.3f}  full {f:7.3f}  done {dn:7.3f}  "
              f"lat {f - (iss[i] - t0) / 1e3:6.3f}  proc {dn - f:6.3f}")
    v = (iss > 0) & (done > 0)
    if v.sum() > 4:
        span = (done[v].max() - iss[v].min()) / 1e3
        print(f"  {v.sum()} blocks in {span:.2f} us: {span / v.sum():.3f} us per block")
e.close()
