"""A/B of the pipelined kernel at the bench config: iteration time with pipe off / on at several
attention-CTA counts (same session inputs).  Usage: python scripts/pipe_ab.py [config]"""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402
import bench  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
c = bench.CONFIGS[name]
L, d, B = c["L"], c["d"], c["B"]
first = np.array([p[-1] for p in bench.workload(B)], np.int32)
for tech in (c["tech"], "never"):
    for pipe, ga in [(0, 0), (1, 84), (1, 92), (1, 100)]:
        cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique(tech),
                             schedule=X.ThresholdSchedule(c["lam"], c["gamma"], 0.0), max_batch=B,
                             pool_blocks=B * L * 40, eos_token=-1)
        e = X.Engine(cfg)
        e.set_option("pipe", pipe)
        if ga:
            e.set_option("pipe_att_ctas", ga)
        e.session_begin(first, 511, 640, 1, np.arange(B))
        e.decode_run(5)
        e.sync()
        ms = e.time_decode(20) / 20
        ex = e.records(5, 20)["output_layer"]
        print(f"{name} {tech:10s} pipe={pipe} att={ga:3d}: {ms * 1e3:8.1f} us/iteration, mean exit {ex.mean():.2f}",
              flush=True)
        e.close()
