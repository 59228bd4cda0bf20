ATTN_AHEAD=0,2,4,8 ATTN_GRIDS=56,92,148 timeout 400 python scripts/attn_grid_probe.py 256 1024 2 3 > gpurun_out/attn_grid3.txt 2>&1
for ah in 0 4 8; do python - <<PY >> gpurun_out/pipe_ahead.txt 2>&1
import sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X
B, L, d = 256, 24, 1024
for ga in (80, 92, 104):
    cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique("never"), max_batch=B, pool_blocks=B * L * 40, eos_token=-1)
    e = X.Engine(cfg, mega=True)
    e.set_option("pipe", 1); e.set_option("pipe_att_ctas", ga); e.set_option("attn_l2_ahead", $ah)
    e.session_begin(np.arange(B) + 1, 511, 640, 1, np.arange(B))
    e.decode_run(2); e.sync()
    ms = e.time_decode(10)
    print(f"ahead $ah att_ctas {ga}: {ms / 10 * 1e3:.1f} us per full-depth iteration")
    e.close()
PY
done
