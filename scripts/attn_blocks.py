"""Per-block timeline of the attention pass (layer 1) for CTAs 0..3 inside the
persistent kernel (dbg 32 stamps: producer issue, consumer start, consumer done).
Usage: python scripts/attn_blocks.py [config] [json options]
Needs the instrumented library: EL_DEBUG=1 python paper_2407_20272_b200/build.py --force
"""
import ctypes as C
import json
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402

DIMS = {"c2": (12, 768, 64), "c3": (24, 1024, 128), "c5": (24, 1024, 256)}
cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
opts = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
L, d, B = DIMS[cfgname]
cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique("never", 4),
                     schedule=X.ThresholdSchedule(0.981, 0.997, 0.0), max_batch=B, pool_blocks=B * L * 40,
                     eos_token=-1)
e = X.Engine(cfg, mega=True)
xdbg = int(opts.pop("xdbg", 0))
for k, v in opts.items():
    e.set_option(k, v)
e.session_begin(np.arange(B) + 1, 511, 640, 1)
lib = X.lib()
lib.el_debug_timestamps.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
e.decode_run(3)
e.sync()
e.set_option("dbg", 32 | 128 | xdbg)
e.decode_run(1)
e.sync()
ts = np.zeros(65536, np.uint64)
lib.el_debug_timestamps(e._h, ts.ctypes.data_as(C.c_void_p), ts.size)
e.set_option("dbg", 0)
A = ts[40000:40000 + 2 * 148].reshape(148, 2).astype(np.float64)  # layer-1 attention spans
t0 = A[:, 0].min()
for cta in range(4):
    iss = ts[8192 + 1024 + cta * 128: 8192 + 1024 + cta * 128 + 60].astype(np.float64)
    got = ts[8192 + cta * 128: 8192 + cta * 128 + 60].astype(np.float64)
    done = ts[8192 + 2048 + cta * 128: 8192 + 2048 + cta * 128 + 60].astype(np.float64)
    n = int(np.argmax(iss == 0)) if (iss == 0).any() else 60
    ck = ts[8192 + 3072 + cta * 16: 8192 + 3072 + cta * 16 + 16].astype(np.float64)
    rel = (ck - ck[0]) / 1965.0
    print(f"CTA {cta}: producer: T/Ts computed {rel[10]:.2f}, split ready {rel[11]:.2f}, first emit before ring wait "
          f"{rel[8]:.2f}, after ring wait {rel[9]:.2f}")
    print(f"CTA {cta}: clocks from phase start (us): producer enters attn_body {rel[1]:.2f}, ids gathered {rel[2]:.2f}, "
          f"first issue {rel[3]:.2f}, consumer first block {rel[4]:.2f}, stream end {rel[5]:.2f}, settled {rel[6]:.2f}")
    print(f"CTA {cta}: span {(A[cta, 0] - t0) / 1e3:.2f} .. {(A[cta, 1] - t0) / 1e3:.2f} us; blocks (issue / consumer start / done, us):")
    row = []
    for k in range(min(n, 40)):
        row.append(f"{(iss[k] - t0) / 1e3:5.2f}/{(got[k] - t0) / 1e3:5.2f}/{(done[k] - t0) / 1e3:5.2f}")
    for k in range(0, len(row), 6):
        print("   " + "  ".join(row[k:k + 6]))
