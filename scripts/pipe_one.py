"""One pipelined iteration at small dims (sanitizer helper)."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402
L, d, V, B = (int(x) for x in sys.argv[1:5])
cfg = X.EngineConfig(model=X.ModelConfig(L, d, V, 0), technique=X.ExitTechnique("classifier"),
                     schedule=X.ThresholdSchedule(0.5, 1.0, 0.0), max_batch=B, pool_blocks=B * L * 8, eos_token=-1)
e = X.Engine(cfg, mega=True)
e.set_option("pipe", 1)
e.session_begin(np.arange(B) % V + 1, 40, 100, 1, np.arange(B))
r = e.decode_iteration()
print("ok exit", r["output_layer"])
