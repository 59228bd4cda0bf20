"""ms/iteration of the bench workload for a list of option sets (device-resident, events)."""
import json, sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X
import bench
cfgname = sys.argv[1]; optsets = json.loads(sys.argv[2])
c = bench.CONFIGS[cfgname]; L, d, B = c["L"], c["d"], c["B"]
prompts = bench.workload(B); first = np.array([p[-1] for p in prompts], np.int32)
for tech in (c["tech"], "never"):
    for opts in optsets:
        cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique(tech),
                             schedule=X.ThresholdSchedule(c["lam"], c["gamma"], 0.0), max_batch=B,
                             pool_blocks=B * L * 40, eos_token=-1)
        e = X.Engine(cfg)
        for k, v in opts.items(): e.set_option(k, v)
        e.session_begin(first, 511, 640, 1, np.arange(B))
        e.decode_run(5); e.sync()
        ms = e.time_decode(30) / 30
        ex = e.records(5, 30)["output_layer"]
        print(json.dumps(dict(cfg=cfgname, tech=tech, opts=opts, ms=round(ms, 4), tok_s=round(B / ms * 1e3), mean_e=float(ex.mean()))), flush=True)
        e.close()
