"""Per-CTA unit timeline of the pipelined kernel's GEMM phases at layer 1 (EL_DEBUG build, dbg 64):
median / max over the GEMM CTAs of each event relative to the phase start (SM clock -> us).
Batch-M phases (QKV, W_o, up): the CTA's last unit of the half-1 pass; split-K down: its unit.
Usage: python scripts/pipe_gemm_tl.py [B] [att_ctas]"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ga = int(sys.argv[2]) if len(sys.argv) > 2 else 92
L, d = 24, 1024
cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique("never"), max_batch=B,
                     pool_blocks=B * L * 40, eos_token=-1)
e = X.Engine(cfg, mega=True)
e.set_option("pipe", 1)
e.set_option("pipe_att_ctas", ga)
e.session_begin(np.arange(B) + 1, 511, 640, 1, np.arange(B))
e.decode_run(2)
e.sync()
e.set_option("dbg", 64)
e.decode_run(1)
e.sync()
lib = X.lib()
lib.el_debug_timestamps.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
ts = np.zeros(320000, np.uint64)
lib.el_debug_timestamps(e._h, ts.ctypes.data_as(C.c_void_p), ts.size)
G = 148
t = ts[300000:300000 + G * 32].reshape(G, 32).astype(np.int64)
clk = 1.965e3  # cycles per us
bm_names = {1: "producer start", 7: "weights ready", 5: "1st act chunk", 6: "last act chunk", 4: "MMAs issued",
            2: "unit done", 3: "epilogue done"}
for K, nm in enumerate(["QKV", "W_o", "up"]):
    rows = t[:, K * 8:(K + 1) * 8]
    v = rows[:, 0] > 0
    print(f"{nm}: {v.sum()} CTAs")
    for k in (1, 7, 5, 6, 4, 2, 3):
        x = (rows[v, k] - rows[v, 0]) / clk
        x = x[rows[v, k] > 0]
        if len(x):
            print(f"   {bm_names[k]:15s} med {np.median(x):7.2f}  max {x.max():7.2f} us")
rows = t[:, 24:32]
v = rows[:, 0] > 0
print(f"down (split-K, fused reduce): {v.sum()} CTAs")
for k, nm in ((6, "1st stage full"), (5, "MMAs issued"), (7, "producer done"), (1, "unit done"), (2, "partial stored"),
              (3, "tile complete"), (4, "reduced")):
    x = (rows[v, k] - rows[v, 0]) / clk
    x = x[rows[v, k] > 0]
    if len(x):
        print(f"   {nm:15s} med {np.median(x):7.2f}  max {x.max():7.2f} us")
e.set_option("dbg", 0)
e.close()
