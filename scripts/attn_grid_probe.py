"""Paged-attention bandwidth vs the number of CTAs streaming it (standalone attn_kernel, cold L2):
how many SMs does the attention pass need to saturate HBM, and how much does one CTA pull?
Usage: python scripts/attn_grid_probe.py [B] [d] [stages...]"""
import json
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
d = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
stages = [int(s) for s in sys.argv[3:]] or [2, 3]
L, prefix = 4, 511
cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique("never"), max_batch=B,
                     pool_blocks=B * L * 40, eos_token=-1)
e = X.Engine(cfg, mega=False)
e.session_begin(np.arange(B) + 1, prefix, 640, 1)
ctx = prefix + 1
a_bytes = B * ctx * 2 * d * 2 + B * d * 4 * 2  # K + V bf16, q fp32 in + out
res = []
import os
if os.environ.get("ATTN_DBG"):  # EL_DEBUG builds: 1 = consumers skip the block math (transfer only)
    e.set_option("dbg", int(os.environ["ATTN_DBG"]))
aheads = [int(x) for x in os.environ.get("ATTN_AHEAD", "4").split(",")]
grids = [int(x) for x in os.environ.get("ATTN_GRIDS", "37,46,56,74,92,110,128,148").split(",")]
for ah in aheads:
    e.set_option("attn_l2_ahead", ah)
    for S in stages:
        e.set_option("attn_stages", S)
        for g in grids:
            e.set_option("attn_grid", g)
            ms = e.time_kernel(0x100, 1, 10)
            gbs = a_bytes / (ms * 1e-3) / 1e9
            res.append({"ahead": ah, "stages": S, "ctas": g, "us": round(ms * 1e3, 2), "GBps": round(gbs, 1),
                        "GBps_per_cta": round(gbs / g, 1)})
            print(json.dumps(res[-1]), flush=True)
e.set_option("attn_grid", 0)
e.close()
