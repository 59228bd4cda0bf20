"""Persistent kernel vs per-phase kernels on the same inputs: hidden state / K,V / tokens after a few iterations."""
import json
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402

L, d, B = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (12, 768, 64)))
opts = json.loads(sys.argv[4]) if len(sys.argv) > 4 else {}
res = []
for mega in (False, True):
    cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique("never"), max_batch=B,
                         pool_blocks=B * L * 42, eos_token=-1)
    e = X.Engine(cfg, mega=mega)
    for k, v in opts.items():
        e.set_option(k, v)
    e.session_begin(np.arange(B) * 7 + 1, 511, 660, 1)
    rs = [e.decode_iteration() for _ in range(2)]
    res.append((rs, e.hidden(L & 1), e.kv(B - 1, 2, 512), e.kv(0, L, 512)))
    e.close()
(ra, ha, ka, kla), (rb, hb, kb, klb) = res
rel = lambda a, b: float(np.abs(a - b).max() / max(np.abs(a).max(), 1e-30))
print("hidden rel", rel(ha, hb), "k(l2) rel", rel(ka[0], kb[0]), "v(l2) rel", rel(ka[1], kb[1]),
      "k(L) rel", rel(kla[0], klb[0]))
print("token agreement", [float(np.mean(x["tokens"] == y["tokens"])) for x, y in zip(ra, rb)])
bad = np.where(np.abs(ha - hb).max(axis=1) > 0.05 * np.abs(ha).max())[0]
print("rows with large hidden error:", bad.tolist()[:40])
