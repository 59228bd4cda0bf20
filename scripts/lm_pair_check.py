"""LM-head variants against each other on a bench workload (B200): every value of the option must
give the same exit layers and tokens (up to exact logit ties), confidences within fp32 reordering
noise.  python scripts/lm_pair_check.py [config c4m] [option lm_pair] [values 0,1,2] [iterations 8]"""
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
from oracle import bindings as OB  # noqa: E402
from paper_2407_20272_b200 import exitlab as X  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4m"
opt = sys.argv[2] if len(sys.argv) > 2 else "lm_pair"
vals = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "0,1,2").split(",")]
N = int(sys.argv[4]) if len(sys.argv) > 4 else 8
c = bench.CONFIGS[name]
L, d, B, V = c["L"], c["d"], c["B"], bench.V
wl = OB.port().gen_workload(n_requests=B, prompt_len_min=512, prompt_len_max=512, output_len_min=128,
                            output_len_max=128, seed=1, vocab_size=V)
first = wl.prompt[wl.prompt_off[1:] - 1]
out = {}
for k in vals:
    cfg = X.EngineConfig(model=X.ModelConfig(L, d, V, 0), technique=X.ExitTechnique(c["tech"]),
                         schedule=X.ThresholdSchedule(c["lam"], c["gamma"], 0.0), max_batch=B,
                         pool_blocks=B * L * 40, eos_token=-1)
    e = X.Engine(cfg)
    e.set_option(opt, k)
    e.session_begin(first, 511, 640, 1)
    e.decode_run(N)
    r = e.records(0, N)
    out[k] = r
    pi = e.plan_info()
    print(name, opt, k, {x: pi.get(x) for x in ("mega", "pipe", "lm_pair", "lm_keep", "lm_tail_tr")},
          "mean e", float(r["output_layer"].mean()), flush=True)
    e.close()
a = out[vals[0]]
for k in vals[1:]:
    b = out[k]
    ca, cb = a["conf"], b["conf"]
    m = np.isfinite(ca) & np.isfinite(cb)
    print(f"{opt} {k} vs {vals[0]}: exit layers equal {np.array_equal(a['output_layer'], b['output_layer'])}, "
          f"tokens equal {(a['tokens'] == b['tokens']).mean():.4f}, max |conf diff| {np.abs(ca[m] - cb[m]).max():.3e}, "
          f"max conf {np.abs(ca[m]).max():.3e}")
