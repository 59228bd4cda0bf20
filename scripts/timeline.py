"""Device-side timeline of one decode iteration (graph or eager): per kernel [start, end] (us)."""
import ctypes as C, json, sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X
tech = sys.argv[1] if len(sys.argv) > 1 else "never"
opts = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
L, d, B = 12, 768, 64
cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique(tech, 4),
                     schedule=X.ThresholdSchedule(0.981, 0.997, 0.0), max_batch=B, pool_blocks=B * L * 40, eos_token=-1)
e = X.Engine(cfg)
for kk, v in opts.items(): e.set_option(kk, v)
e.set_option("dbg", 64)
e.session_begin(np.arange(B) + 1, 511, 640, 1)
lib = X.lib()
lib.el_debug_timestamps.argtypes = [C.c_void_p, C.c_void_p, C.c_int]; lib.el_debug_timeline_reset.argtypes = [C.c_void_p]
e.decode_run(3); e.sync()
lib.el_debug_timeline_reset(e._h)
e.decode_run(1); e.sync()
ts = np.zeros(65536, np.uint64); lib.el_debug_timestamps(e._h, ts.ctypes.data_as(C.c_void_p), 65536)
t = ts[16384:16384 + 2 * 32 * 16].reshape(16, 32, 2).astype(np.float64)
names = {11: "head", 0: "embed", 1: "qkv", 2: "attn", 3: "wo", 4: "up", 5: "down", 10: "lmchk", 6: "exit", 7: "fill", 8: "lm", 9: "finish"}
valid = t[:, :, 0] < 1.8e19
t0 = t[:, :, 0][valid].min()
ev = []
for kind, nm in names.items():
    for layer in range(32):
        if valid[kind, layer]:
            ev.append((t[kind, layer, 0] - t0, t[kind, layer, 1] - t0, nm, layer))
ev.sort()
prev_end = 0.0
busy = 0.0
for s, en, nm, layer in ev:
    print(f"{nm:7s} L{layer:2d} start {s/1e3:8.2f} end {en/1e3:8.2f} dur {(en-s)/1e3:6.2f} gap {(s-prev_end)/1e3:6.2f}")
    busy += en - s
    prev_end = max(prev_end, en)
print(f"iteration span {prev_end/1e3:.2f} us, sum of kernel spans {busy/1e3:.2f} us")
