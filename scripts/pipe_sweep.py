"""Full-depth iteration time of the pipelined kernel (c5 dims) over engine options, same box:
    python scripts/pipe_sweep.py '[{"pipe_att_ctas": 92}, {"pipe_att_ctas": 100, "mega_bm_wstream": 0}]'
(used for the attention-CTA count, batch-M slab / streamed weights and chunk-size choices)."""
import json
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402

B, L, d = 256, 24, 1024
for opts in json.loads(sys.argv[1]) if len(sys.argv) > 1 else [{}]:
    cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique("never"), max_batch=B,
                         pool_blocks=B * L * 40, eos_token=-1)
    e = X.Engine(cfg, mega=True)
    e.set_option("pipe", 1)
    for k, v in opts.items():
        e.set_option(k, v)
    e.session_begin(np.arange(B) + 1, 511, 640, 1, np.arange(B))
    e.decode_run(2)
    e.sync()
    ms = min(e.time_decode(10) for _ in range(3))
    print(f"{json.dumps(opts)}: {ms / 10 * 1e3:.1f} us per full-depth iteration", flush=True)
    e.close()
