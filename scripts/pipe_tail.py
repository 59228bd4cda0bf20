"""Tail of the pipelined kernel (EL_DEBUG build, dbg 128): after the layer loop, the LM head +
skipped-layer fill units, the barrier, the fill reduce and the greedy token, at the bench's
early exit (c5 classifier) -- per-phase microseconds of CTA 0.  Usage: python scripts/pipe_tail.py"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402

B, L, d = 256, 24, 1024
cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique("classifier"),
                     schedule=X.ThresholdSchedule(0.41, 0.997, 0.0), max_batch=B, pool_blocks=B * L * 42,
                     eos_token=-1)
e = X.Engine(cfg, mega=True)
e.session_begin(np.arange(B) + 1, 511, 660, 1, np.arange(B))
e.decode_run(3)
e.sync()
lib = X.lib()
lib.el_debug_timestamps.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
for it in range(3):
    e.set_option("dbg", 128)
    r = e.decode_iteration()
    e.set_option("dbg", 0)
    ts = np.zeros(201064, np.uint64)
    lib.el_debug_timestamps(e._h, ts.ctypes.data_as(C.c_void_p), ts.size)
    t = ts[200000:200800].reshape(25, 2, 16).astype(np.float64)
    tail = t[24, 0, :4]
    st0, emb = t[24, 1, 0], t[24, 1, 1]
    l1 = t[0, 0, 0]  # attention CTA 0 starts layer 1 (QKV(H0, 1) published)
    per_layer = [(t[l, 1, 6] - t[l - 1, 1, 6]) / 1e3 for l in range(1, 24) if t[l, 1, 6] and t[l - 1, 1, 6]]
    print(f"  start -> embed done {(emb - st0) / 1e3:.1f} us -> first attention {(l1 - emb) / 1e3:.1f} us | layers "
          f"{len(per_layer)} x {np.mean(per_layer) if per_layer else 0:.1f} us | total {(tail[3] - st0) / 1e3:.1f} us")
    ex = r["output_layer"]
    last = t[ex - 1, 1, 5] if t[ex - 1, 1, 5] else t[ex - 1, 1, :7].max()
    print(f"exit {ex}: loop end -> tail start {(tail[0] - last) / 1e3:.1f} us | LM + fill units {(tail[1] - tail[0]) / 1e3:.1f}"
          f" | barrier {(tail[2] - tail[1]) / 1e3:.1f} | fill reduce + greedy {(tail[3] - tail[2]) / 1e3:.1f} us")

    u = ts[201000:201064].reshape(2, 8, 4).astype(np.float64)
    for c in range(2):
        rows = [r for r in u[c] if r[0] > 0]
        print(f"   cta {c}: " + " | ".join(f"unit {i}: load+mma {(r[1] - r[0]) / 1e3:.1f} epi {(r[2] - r[1]) / 1e3:.1f}"
                                         for i, r in enumerate(rows)))
