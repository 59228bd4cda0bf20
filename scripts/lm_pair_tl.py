"""Timeline of the softmax check's LM pair units at layer 1 (EL_DEBUG=1 build; dbg bit 64):
per CTA, clock64 from the LM loop start to the first / last stage full, producer done, accumulator
ready and epilogue done of its first unit (p50 / max over CTAs, us at 1.965 GHz).
    python scripts/lm_pair_tl.py [c3|c2] [json options]"""
import ctypes as C
import json
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402

DIMS = {"c2": (12, 768, 64), "c3": (24, 1024, 128)}
L, d, B = DIMS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
opts = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique("softmax", 4),
                     schedule=X.ThresholdSchedule(0.981, 0.997, 0.0), max_batch=B, pool_blocks=B * L * 40,
                     eos_token=-1)
e = X.Engine(cfg, mega=True)
for k, v in opts.items():
    e.set_option(k, v)
e.session_begin(np.arange(B) + 1, 511, 640, 1)
lib = X.lib()
lib.el_debug_timestamps.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
e.decode_run(3)
e.sync()
e.set_option("dbg", 64)
e.decode_run(1)
e.sync()
ts = np.zeros(65536 + 256 * 1024, np.uint64)
lib.el_debug_timestamps(e._h, ts.ctypes.data_as(C.c_void_p), ts.size)
a = ts[320000:320000 + 148 * 8].reshape(148, 8).astype(np.float64)
a = a[a[:, 6] > 0]
rel = (a - a[:, :1]) / 1965.0
print(f"{len(a)} CTAs with an LM unit; plan {e.plan_info()}")
for k, nm in ((1, "first stage full"), (2, "last stage full"), (4, "producer done"), (5, "acc ready"),
              (6, "epilogue done")):
    print(f"{nm:18s} p50 {np.median(rel[:, k]):7.2f}  max {rel[:, k].max():7.2f} us")
