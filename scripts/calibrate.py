"""Mean exit layer of the bench workload under a grid of threshold schedules (B200).

    python scripts/calibrate.py L d B tech '[[lam, gamma], ...]' [iterations (16)]
"""
import json, sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X
from oracle import bindings as OB
L, d, B, tech = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
grid = json.loads(sys.argv[5])
N = int(sys.argv[6]) if len(sys.argv) > 6 else 16
V = 32128
wl = OB.port().gen_workload(n_requests=B, prompt_len_min=512, prompt_len_max=512, output_len_min=128,
                            output_len_max=128, seed=1, vocab_size=V)
first = wl.prompt[wl.prompt_off[1:] - 1]
for lam, gam in grid:
    cfg = X.EngineConfig(model=X.ModelConfig(L, d, V, 0), technique=X.ExitTechnique(tech),
                         schedule=X.ThresholdSchedule(lam, gam, 0.0), max_batch=B, pool_blocks=B * L * 40, eos_token=-1)
    e = X.Engine(cfg)
    e.session_begin(first, 511, 640, 1)
    e.decode_run(N)
    r = e.records(0, N)
    c = r["conf"]  # [it][L][B]
    print(json.dumps(dict(lam=lam, gamma=gam, mean_e=float(r["output_layer"].mean()), e=r["output_layer"].tolist(),
                          conf_p50_by_layer=[float(np.nanmedian(c[:, l, :])) for l in range(L)][:6],
                          conf_min_l1=float(np.nanmin(c[:, 0, :])))), flush=True)
    e.close()
