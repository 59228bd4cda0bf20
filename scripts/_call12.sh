python - <<'PY' > gpurun_out/pipe_slab.txt 2>&1
import sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X
B, L, d = 256, 24, 1024
for slab, ck, ga in ((96, 32, 92), (96, 64, 92), (128, 32, 92), (128, 32, 84), (128, 32, 100), (112, 32, 92), (160, 16, 92)):
    cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique("never"), max_batch=B, pool_blocks=B * L * 40, eos_token=-1)
    e = X.Engine(cfg, mega=True)
    e.set_option("pipe", 1); e.set_option("mega_bm_chunk_kb", ck); e.set_option("pipe_slab_kb", slab); e.set_option("pipe_att_ctas", ga)
    try:
        e.session_begin(np.arange(B) + 1, 511, 640, 1, np.arange(B))
        e.decode_run(2); e.sync()
        ms = e.time_decode(10)
        print(f"slab {slab} KB chunk {ck} KB att {ga}: {ms / 10 * 1e3:.1f} us per full-depth iteration {e.plan_info()}", flush=True)
    except Exception as ex:
        print(f"slab {slab} chunk {ck}: {ex}", flush=True)
    e.close()
PY
