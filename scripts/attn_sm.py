"""Per-SM attention pass durations inside the persistent kernel (dbg 128 stamps):
which SMs are slow, is it stable across layers / iterations, and does it follow
the GPC / die layout?  Usage: python scripts/attn_sm.py [config] [json options]
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
durs = []
smid = None
for it in range(6):
    e.set_option("dbg", 128 | xdbg)
    e.decode_run(1)
    e.sync()
    ts = np.zeros(65536 + 256 * 1024, np.uint64)
    lib.el_debug_timestamps(e._h, ts.ctypes.data_as(C.c_void_p), ts.size)
    A = ts[40000:40000 + 24 * 512].reshape(24, 256, 2).astype(np.float64)[:L, :148]
    smid = ts[40000 + 24 * 512:40000 + 24 * 512 + 148].astype(np.int64)
    st = A[:, :, 0].min(axis=1, keepdims=True)
    durs.append((A[:, :, 1] - A[:, :, 0]) / 1e3)  # [layer][cta]
e.set_option("dbg", xdbg)
print(f"timed: {e.time_decode(20) / 20 * 1e3:.1f} us/iteration (options {opts}, dbg {xdbg})")
e.set_option("dbg", 0)
D = np.stack(durs)  # [it][layer][cta]
per_cta = D.mean(axis=(0, 1))
print(f"config {cfgname}: attention pass per CTA: mean {per_cta.mean():.2f} min {per_cta.min():.2f} max {per_cta.max():.2f} us")
# stability: correlation of per-CTA durations between iterations / layers
flat = D.reshape(-1, 148)
cc = np.corrcoef(flat)
print(f"correlation of per-CTA duration vectors across (iteration, layer) samples: mean {cc[np.triu_indices_from(cc, 1)].mean():.3f}")
by_sm = np.full(148, np.nan)
by_sm[smid] = per_cta
print("per-SM mean duration (us), rows of 16 SM ids:")
for r in range(0, 148, 16):
    print(f"  sm {r:3d}: " + " ".join(f"{x:5.1f}" for x in by_sm[r:r + 16]))
# TPC (SM pair) and die halves
print(f"SM 0-73 mean {np.nanmean(by_sm[:74]):.2f}, SM 74-147 mean {np.nanmean(by_sm[74:]):.2f}")
print(f"even SMs {np.nanmean(by_sm[0::2]):.2f}, odd SMs {np.nanmean(by_sm[1::2]):.2f}")
# work structure of the static split: segments per CTA and row ends (combine candidates)
pos = int(e.plan_info().get("pos0", 0)) if False else None
bc = 16
for nb in sorted({(p + bc) // bc for p in range(511, 530)}):
    T = B * nb
    seg = np.zeros(148, int)
    ends = np.zeros(148, int)
    for i in range(148):
        g0, g1 = i * T // 148, (i + 1) * T // 148
        rows = set(range(g0 // nb, (g1 - 1) // nb + 1)) if g1 > g0 else set()
        seg[i] = len(rows)
        ends[i] = sum(1 for r in rows if (r + 1) * nb - 1 < g1)
    for k in sorted(set(seg)):
        m = seg == k
        print(f"  nb={nb}: CTAs with {k} segments: n={m.sum():3d} mean dur {per_cta[m].mean():.2f} us")
    for k in sorted(set(ends)):
        m = ends == k
        print(f"  nb={nb}: CTAs with {k} row ends: n={m.sum():3d} mean dur {per_cta[m].mean():.2f} us")
np.save("gpurun_out/attn_sm.npy", np.stack([np.arange(148), by_sm]))
