python - <<'PY' > gpurun_out/pipe_slab2.txt 2>&1
import sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X
B, L, d = 256, 24, 1024
for slab, ck, ga in ((96, 32, 92), (128, 32, 96), (128, 32, 100), (128, 32, 104), (128, 32, 108), (128, 32, 112), (96, 32, 92), (128, 32, 100)):
    cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique("never"), max_batch=B, pool_blocks=B * L * 40, eos_token=-1)
    e = X.Engine(cfg, mega=True)
    e.set_option("pipe", 1); e.set_option("mega_bm_chunk_kb", ck); e.set_option("pipe_slab_kb", slab); e.set_option("pipe_att_ctas", ga)
    e.session_begin(np.arange(B) + 1, 511, 640, 1, np.arange(B))
    e.decode_run(2); e.sync()
    ms = min(e.time_decode(10) for _ in range(3))
    print(f"slab {slab} KB chunk {ck} KB att {ga}: {ms / 10 * 1e3:.1f} us per full-depth iteration", flush=True)
    e.close()
PY
