"""A/B of streamed batch-M weights (mega_bm_wstream) on the persistent / pipelined kernels: full-depth
iteration time and bitwise equality of the hidden state.  Usage: python scripts/wstream_ab.py"""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X  # noqa: E402

CASES = [("c5 pipe", 24, 1024, 256, {"pipe": 1}, [92, 100, 108, 116]),
         ("c3 iter", 24, 1024, 128, {}, [0]), ("c2 iter", 12, 768, 64, {}, [0])]
for name, L, d, B, opts, gas in CASES:
    for ga in gas:
        ref = None
        for ws in (0, 1):
            cfg = X.EngineConfig(model=X.ModelConfig(L, d, 32128, 0), technique=X.ExitTechnique("never"), max_batch=B,
                                 pool_blocks=B * L * 40, eos_token=-1)
            e = X.Engine(cfg, mega=True)
            for k, v in opts.items():
                e.set_option(k, v)
            if ga:
                e.set_option("pipe_att_ctas", ga)
            e.set_option("mega_bm_wstream", ws)
            e.session_begin(np.arange(B) + 1, 511, 640, 1, np.arange(B))
            e.decode_run(2)
            e.sync()
            h = e.hidden(L & 1).copy()
            ms = min(e.time_decode(10) for _ in range(3))
            same = "" if ref is None else f" hidden bit-identical to ws=0: {bool(np.array_equal(h, ref))}"
            ref = h if ref is None else ref
            print(f"{name} att {ga} wstream {ws}: {ms / 10 * 1e3:.1f} us per full-depth iteration{same}", flush=True)
            e.close()
