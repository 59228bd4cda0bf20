for ck in 16 32 64; do python - <<PY >> gpurun_out/pipe_chunk.txt 2>&1
import sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X
B, L, d = 256, 24, 1024
cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique("never"), max_batch=B, pool_blocks=B * L * 40, eos_token=-1)
e = X.Engine(cfg, mega=True)
e.set_option("pipe", 1); e.set_option("mega_bm_chunk_kb", $ck)
e.session_begin(np.arange(B) + 1, 511, 640, 1, np.arange(B))
e.decode_run(2); e.sync()
ms = e.time_decode(10)
print(f"chunk $ck KB: {ms / 10 * 1e3:.1f} us per full-depth iteration")
PY
done
EL_DEBUG=1 python paper_2407_20272_b200/build.py --force > gpurun_out/dbg_build.txt 2>&1
timeout 300 python scripts/mega_phases.py c1 softmax '{"mega": 1}' > gpurun_out/mega_c1.txt 2>&1
timeout 300 python scripts/mega_phases.py c1 never > gpurun_out/mega_c1_never.txt 2>&1
