"""Timeline of the pipelined kernel (EL_DEBUG=1 build): per (layer, half) the attention pass of
attention CTA 0 and the GEMM chain of GEMM CTA GA, in us from the first stamp.
Usage: python scripts/pipe_timeline.py [B] [att_ctas] [layers to show]"""
import ctypes as C
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402
B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ga = int(sys.argv[2]) if len(sys.argv) > 2 else 84
show = int(sys.argv[3]) if len(sys.argv) > 3 else 4
L, d = 24, 1024
cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique("never"),
                     max_batch=B, pool_blocks=B * L * 40, eos_token=-1)
e = X.Engine(cfg, mega=True)
e.set_option("pipe", 1)
e.set_option("pipe_att_ctas", ga)
e.session_begin(np.arange(B) + 1, 511, 640, 1, np.arange(B))
e.decode_run(2)
e.sync()
e.set_option("dbg", 128)
e.decode_run(1)
e.sync()
lib = X.lib()
lib.el_debug_timestamps.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
ts = np.zeros(200000 + 24 * 2 * 16, np.uint64)
lib.el_debug_timestamps(e._h, ts.ctypes.data_as(C.c_void_p), ts.size)
t = ts[200000:].reshape(24, 2, 16).astype(np.float64)
t0 = t[t > 0].min()
names = ["att wait done", "att pass done", "gemm: att ready", "W_o", "up", "down", "QKV next"]
for layer in range(min(show, L)):
    for h in range(2):
        row = t[layer, h, :7]
        print(f"L{layer + 1} H{h}: " + " | ".join(f"{n} {(v - t0) / 1e3:7.2f}" for n, v in zip(names, row) if v > 0))
e.set_option("dbg", 0)
ms = e.time_decode(10)
print(f"att {ga}: {ms / 10 * 1e3:.1f} us/iteration ({(t[L - 1, 1, 1] - t0) / 1e3 / L if t[L - 1, 1, 1] else 0:.1f} us/layer)")
