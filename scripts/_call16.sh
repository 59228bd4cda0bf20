python - <<'PY' > gpurun_out/bmdown.txt 2>&1
import sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X
B, L, d = 256, 24, 1024
for bd, ga in ((0, 100), (1, 100), (1, 96), (1, 92), (1, 104), (0, 100), (1, 100)):
    cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique("never"), max_batch=B, pool_blocks=B * L * 40, eos_token=-1)
    e = X.Engine(cfg, mega=True)
    e.set_option("pipe", 1); e.set_option("pipe_att_ctas", ga); e.set_option("pipe_bm_down", bd)
    e.session_begin(np.arange(B) + 1, 511, 640, 1, np.arange(B))
    e.decode_run(2); e.sync()
    h = e.hidden(L & 1).copy()
    ms = min(e.time_decode(10) for _ in range(3))
    print(f"bm_down {bd} att {ga}: {ms / 10 * 1e3:.1f} us per full-depth iteration, |h| {np.abs(h).max():.4f} h[0,:3] {h[0,:3]}", flush=True)
    e.close()
PY
