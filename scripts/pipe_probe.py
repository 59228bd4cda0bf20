"""Pipelined kernel vs the plain persistent kernel: same session, tokens / exits / hidden states,
and iteration time (debug helper).  Usage: python scripts/pipe_probe.py [B] [att_ctas] [tech]"""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402
import bench  # noqa: E402
B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ga = int(sys.argv[2]) if len(sys.argv) > 2 else 84
tech = sys.argv[3] if len(sys.argv) > 3 else "classifier"
c = bench.CONFIGS["c5"]
L, d = c["L"], c["d"]
first = np.array([p[-1] for p in bench.workload(B)], np.int32)
out = {}
for pipe in (0, 1):
    cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique(tech),
                         schedule=X.ThresholdSchedule(c["lam"] if tech == "classifier" else 0.9819,
                                                      c["gamma"] if tech == "classifier" else 0.999, 0.0),
                         max_batch=B, pool_blocks=B * L * 40, eos_token=-1)
    e = X.Engine(cfg, mega=True)
    e.set_option("pipe", pipe)
    e.set_option("pipe_att_ctas", ga)
    e.session_begin(first, 511, 640, 1, np.arange(B))
    rs = [e.decode_iteration() for _ in range(3)]
    h = e.hidden(rs[-1]["output_layer"] & 1)
    ms = e.time_decode(20) / 20
    out[pipe] = (rs, h, ms)
    print(f"pipe={pipe}: exits {[r['output_layer'] for r in rs]} {ms * 1e3:.1f} us/iteration", flush=True)
    e.close()
(ra, ha, _), (rb, hb, _) = out[0], out[1]
for x, y in zip(ra, rb):
    print("same exit", x["output_layer"] == y["output_layer"], "tokens agree", float(np.mean(x["tokens"] == y["tokens"])),
          "accept agree", float(np.mean(x["accept"] == y["accept"])))
print("h max abs diff", float(np.abs(ha - hb).max()), "bitwise", bool(np.array_equal(ha, hb)))
