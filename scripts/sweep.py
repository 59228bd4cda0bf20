"""Timing sweep of plan options at a bench config (device-resident, CUDA events)."""
import argparse, itertools, json, sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X

ap = argparse.ArgumentParser()
ap.add_argument("--L", type=int, default=12); ap.add_argument("--d", type=int, default=768)
ap.add_argument("--B", type=int, default=64); ap.add_argument("--tech", default="never")
ap.add_argument("--exit_layer", type=int, default=1)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--opts", default='[{}]')
a = ap.parse_args()
V = 32128
cfg = X.EngineConfig(model=X.ModelConfig(a.L, a.d, V, 0), technique=X.ExitTechnique(a.tech, a.exit_layer),
                     schedule=X.ThresholdSchedule(0.972, 0.998, 0.0), max_batch=a.B, pool_blocks=a.B * a.L * 40,
                     eos_token=-1)
e = X.Engine(cfg)
rng = np.random.default_rng(1)
first = rng.integers(1, V, a.B)
for opt in json.loads(a.opts):
    for k, v in opt.items():
        e.set_option(k, v)
    e.session_begin(first, 511, 640, 1)
    e.decode_run(3); e.sync()
    ms = e.time_decode(a.iters) / a.iters
    rec = e.records(3, a.iters)
    kt = {name: round(e.time_kernel(kind, 1, 20) * 1e3, 1) for kind, name in
          [(0, "attn"), (1, "qkv"), (2, "wo"), (3, "up"), (4, "down"), (5, "lm")]}
    print(json.dumps(dict(opt=opt, ms_per_iter=round(ms, 4), tok_s=round(a.B / ms * 1e3),
                          mean_e=float(rec["output_layer"].mean()), kernels_us=kt, plan=e.plan_info())), flush=True)
    e.session_end()
