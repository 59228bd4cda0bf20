"""Per-layer cost in graph mode: time always_at(k) iterations for several k and fit a + b*k."""
import json, sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X
L, d, B = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (12, 768, 64)
opts = json.loads(sys.argv[4]) if len(sys.argv) > 4 else {}
V = 32128
ks = [1, 2, 4, 8, L]
res = []
for k in ks:
    cfg = X.EngineConfig(model=X.ModelConfig(L, d, V, 0), technique=X.ExitTechnique.always_at(k), max_batch=B,
                         pool_blocks=B * L * 40, eos_token=-1)
    e = X.Engine(cfg)
    for kk, v in opts.items():
        e.set_option(kk, v)
    e.session_begin(np.arange(B) + 1, 511, 640, 1)
    e.decode_run(3); e.sync()
    ms = e.time_decode(20) / 20
    kt = {name: round(e.time_kernel(kind, 1, 10) * 1e3, 1) for kind, name in
          [(0, "attn"), (1, "qkv"), (2, "wo"), (3, "up"), (4, "down"), (5, "lm")]} if k == 1 else None
    res.append(ms)
    print(json.dumps(dict(k=k, ms=round(ms, 4), kernels_us=kt)), flush=True)
    e.close()
b, a = np.polyfit(ks, res, 1)
print(json.dumps(dict(per_layer_us=round(b * 1e3, 2), fixed_us=round(a * 1e3, 2), opts=opts)))
