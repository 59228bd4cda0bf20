"""Phase timeline of the persistent decode-iteration kernel (dbg bit 128: CTA 0
stamps %globaltimer at every grid barrier).  Usage:
    python scripts/mega_phases.py [config c2|c5|c1|c3] [technique] [json options]
Prints per-phase durations of one iteration, averaged per layer.
Needs the instrumented library: EL_DEBUG=1 python paper_2407_20272_b200/build.py --force
"""
import ctypes as C
import json
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402

DIMS = {"c1": (6, 512, 8), "c2": (12, 768, 64), "c3": (24, 1024, 128), "c5": (24, 1024, 256)}
cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
tech = sys.argv[2] if len(sys.argv) > 2 else "never"
opts = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {}
L, d, B = DIMS[cfgname]
cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique(tech, 4),
                     schedule=X.ThresholdSchedule(0.981, 0.997, 0.0), max_batch=B, pool_blocks=B * L * 40,
                     eos_token=-1)
e = X.Engine(cfg, mega=True)
for kk, v in opts.items():
    if kk != "xdbg":
        e.set_option(kk, v)
e.session_begin(np.arange(B) + 1, 511, 640, 1)
lib = X.lib()
lib.el_debug_timestamps.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
e.decode_run(3)
e.sync()
e.set_option("dbg", 128 | 64 | int(opts.get("xdbg", 0)))
e.decode_run(1)
e.sync()
ts = np.zeros(65536 + 256 * 1024, np.uint64)
lib.el_debug_timestamps(e._h, ts.ctypes.data_as(C.c_void_p), ts.size)
t = ts[20480:20480 + 1024].astype(np.float64)
n = int(np.argmax(t == 0)) if (t == 0).any() else 1024
t = t[:n]
dt = np.diff(t) / 1e3
pi = e.plan_info()
per_layer = []
for nm in ("qkv", "attn", "wo", "up", "down"):
    per_layer.append(nm)
print({k: v for k, v in pi.items() if k.startswith("mega")})
if tech == "softmax":
    per_layer += ["lmchk", "sm_decide"]
names = ["embed->first"]
rec = e.records(3, 1)
eo = int(rec["output_layer"][0])
for layer in range(eo):
    names += [f"{x}@{layer + 1}" for x in per_layer]
names += ["tail(lm+fill)"]
print(f"config {cfgname} tech {tech} e={eo} barriers={n} span {(t[-1] - t[0]) / 1e3:.2f} us")
acc = {}
arr = ts[65536:65536 + 148 * 1024].reshape(148, 1024)[:, :n].astype(np.float64)  # per-CTA arrival times
wrk = {}
for i, v in enumerate(dt):
    nm = names[i + 1] if i + 1 < len(names) else f"?{i}"
    key = nm.split("@")[0]
    acc.setdefault(key, []).append(v)
    # critical path of the phase: last CTA arrival - previous barrier exit (CTA 0)
    wrk.setdefault(key, []).append((arr[:, i + 1].max() - t[i]) / 1e3)
for k, v in acc.items():
    print(f"{k:12s} n={len(v):3d} mean {np.mean(v):7.2f} us  (work crit path {np.mean(wrk[k]):6.2f}, barrier "
          f"{np.mean(v) - np.mean(wrk[k]):5.2f})  total {np.sum(v):8.2f} us")
e.set_option("dbg", 0)
ms = e.time_decode(10)
print(f"timed: {ms / 10 * 1e3:.1f} us/iteration")
# per-CTA attention phase spans (dbg 128): start skew and duration spread
A = ts[40000:40000 + 24 * 512].reshape(24, 256, 2).astype(np.float64)[:, :148]
for layer in (0, eo - 1):
    a = A[layer]
    if a[:, 0].min() == 0:
        continue
    st0 = a[:, 0].min()
    dur = (a[:, 1] - a[:, 0]) / 1e3
    print(f"attn layer {layer + 1}: start skew {(a[:, 0].max() - st0) / 1e3:.2f} us, dur min {dur.min():.2f} "
          f"p50 {np.median(dur):.2f} max {dur.max():.2f} us, last end {(a[:, 1].max() - st0) / 1e3:.2f} us")
    order = np.argsort(dur)
    print("   slowest CTAs:", order[-8:].tolist(), "fastest:", order[:8].tolist())

# batch-M GEMM unit timeline of layer 1 (dbg 64), SM clock cycles:
# [0 start, 1 producer issues, 2 acc ready, 3 epilogue done, 4 MMA issue done, 5 chunk0 full, 6 last chunk full,
#  7 weights ready]
U = ts[300000:300000 + 148 * 32].reshape(148, 4, 8).astype(np.float64)
MHZ = 1965.0
for k, nm in ((0, "qkv"), (1, "wo"), (2, "up")):
    u = U[:, k]
    ok = (u[:, 0] > 0) & (u[:, 2] > 0)
    if not ok.any():
        continue
    rel = lambda j: (u[ok, j] - u[ok, 0]) / MHZ
    print(f"{nm:4s} (n={ok.sum():3d} CTAs, us from phase start, p50/max): producer issue {np.median(rel(1)):.2f}/{rel(1).max():.2f}"
          f" | weights {np.median(rel(7)):.2f}/{rel(7).max():.2f} | chunk0 {np.median(rel(5)):.2f}/{rel(5).max():.2f}"
          f" | last chunk {np.median(rel(6)):.2f}/{rel(6).max():.2f} | MMA issued {np.median(rel(4)):.2f}/{rel(4).max():.2f}"
          f" | acc {np.median(rel(2)):.2f}/{rel(2).max():.2f} | epilogue done {np.median(rel(3)):.2f}/{rel(3).max():.2f}")
u = U[:, 3]
ok = (u[:, 0] > 0) & (u[:, 4] > 0)
if ok.any():
    rel = lambda j: (u[ok, j] - u[ok, 0]) / MHZ
    print(f"down (fused split-K, n={ok.sum()} CTAs with a unit, us p50/max): acc ready {np.median(rel(1)):.2f}/{rel(1).max():.2f}"
          f" | partial stored {np.median(rel(2)):.2f}/{rel(2).max():.2f} | tile complete {np.median(rel(3)):.2f}/{rel(3).max():.2f}"
          f" | reduced {np.median(rel(4)):.2f}/{rel(4).max():.2f}")
    print(f"     mainloop: first stage full {np.median(rel(5)):.2f}/{rel(5).max():.2f} | last stage full "
          f"{np.median(rel(6)):.2f}/{rel(6).max():.2f} | producer done {np.median(rel(7)):.2f}/{rel(7).max():.2f}")
R = ts[310000:310000 + 148 * 8].reshape(148, 8).astype(np.float64)
okr = R[:, 0] > 0
if okr.any():
    rr = lambda j: (R[okr, j] - R[okr, 0]) / MHZ
    print(f"down reduce (warp 0, us from reduce start p50/max): side loads issued {np.median(rr(1)):.2f}/{rr(1).max():.2f}"
          f" | partials summed {np.median(rr(2)):.2f}/{rr(2).max():.2f} | h stored {np.median(rr(3)):.2f}/{rr(3).max():.2f}"
          f" | exit dots {np.median(rr(4)):.2f}/{rr(4).max():.2f}")
okf = (R[:, 5] > 0) & (U[:, 3, 0] > 0)
if okf.any():
    rel5 = (R[okf, 5] - U[okf, 3, 0]) / MHZ
    print(f"down: arrival (red.release) done p50/max {np.median(rel5):.2f}/{rel5.max():.2f} us from phase start")
