import sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X
for L, B in ((2, 128), (2, 96), (4, 128), (4, 72)):
    hs = {}
    for k in (0, 1):
        cfg = X.EngineConfig(model=X.ModelConfig(L, 1024, 32128, 0), technique=X.ExitTechnique("never"),
                             max_batch=128, pool_blocks=128 * L * 42, eos_token=-1)
        e = X.Engine(cfg, mega=True)
        e.set_option("pipe128", k)
        e.session_begin(np.arange(B) + 1, 511, 660, 1)
        r = e.decode_iteration()
        hs[k] = (e.hidden(r["output_layer"] & 1).copy(), r["tokens"].copy(), e.plan_info()["pipe"])
        e.close()
    d = np.abs(hs[0][0] - hs[1][0]).max(axis=1) / np.abs(hs[0][0]).max()
    print(L, B, "pipe", hs[1][2], "rows 0-63 max rel", d[:64].max(), "rows 64+", d[64:B].max(),
          "worst rows", np.argsort(-d)[:8].tolist(), "tokens equal", (hs[0][1] == hs[1][1]).mean(), flush=True)
