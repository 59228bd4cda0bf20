"""Regenerate tests/golden/*.json from the REFERENCE ITSELF.

Runs only where /root/reference exists (this container): it loads
oracle/_ref/libexitlab_ref.so -- the unmodified reference sources compiled in
place -- and records its outputs.  The fixtures are committed; the CPU tests
check the C restatement (oracle/liboracle.so) against them bit for bit, so the
oracle stays pinned on machines without /root/reference (the GPU box).

Floats are stored with float.hex() so the comparison is exact.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import bindings as B  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def hx(a):
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).ravel()]


def main():
    B.build()
    R = B.ref()
    assert R is not None, "reference not built"

    # 1. seeded weights (ModelWeights::seeded, model.cpp:37-59), full tensors of a tiny model
    m = R.model(3, 8, 16, 11)
    weights = {"config": [3, 8, 16, 11], "tensors": {}}
    for name in ["embedding", "lm_head", "probe_w", "probe_b"]:
        weights["tensors"][name] = hx(m.tensor(name))
    for layer in (1, 2, 3):
        for name in ["w_q", "w_k", "w_v", "w_o", "w_up", "w_down"]:
            weights["tensors"][f"{name}@{layer}"] = hx(m.tensor(name, layer))
    # plus checksums of an acceptance-scale model and a BASELINE-scale slice
    m2 = R.model(8, 64, 256, 1000)
    weights["checks"] = {
        "L8d64V256s1000": {n: hx([m2.tensor(n, 1).sum(), m2.tensor(n, 1).ravel()[7]])
                           for n in ["w_q", "w_k", "w_v", "w_o", "w_up", "w_down"]}}
    with open(os.path.join(OUT, "weights.json"), "w") as f:
        json.dump(weights, f)

    # 2. known answers of the exit criteria (exit_policy.cpp:57-87) and threshold_at
    rng = np.random.default_rng(3)
    ka = {"softmax": [], "state": [], "classifier": [], "threshold": []}
    for logits in ([10.0, 0.0, 0.0], [1.0, 1.0, 1.0], [5.0, 5.0, 0.0], rng.normal(size=32).tolist(),
                   (rng.normal(size=1000) * 0.01).tolist()):
        ka["softmax"].append({"in": hx(logits), "out": float(R.softmax_response(logits)).hex()})
    for _ in range(5):
        u, v = rng.normal(size=16), rng.normal(size=16)
        ka["state"].append({"u": hx(u), "v": hx(v), "out": float(R.state_similarity(u, v)).hex()})
        h, w, b = rng.normal(size=16), rng.normal(size=16), float(rng.normal())
        ka["classifier"].append({"h": hx(h), "w": hx(w), "b": b.hex(), "out": float(R.classifier(h, w, b)).hex()})
    for sched in ((0.85, 1.0, 0.0), (0.9, 0.9, 0.0), (0.9, 0.5, 0.4), (0.97, 0.995, 0.0)):
        ka["threshold"].append({"s": list(sched), "out": [float(R.threshold_at(*sched, l)).hex() for l in range(1, 25)]})
    with open(os.path.join(OUT, "known_answers.json"), "w") as f:
        json.dump(ka, f)

    # 3. ExitStatusVector traces (engine.cpp:47-75) on random confidence matrices
    traces = []
    for t in range(200):
        Bsz, L = int(rng.integers(1, 9)), int(rng.integers(2, 11))
        conf = rng.random((L, Bsz))
        lam = rng.random(L) * 0.5 + 0.5
        out, fa = R.status_trace(conf, lam)
        traces.append({"conf": hx(conf), "L": L, "B": Bsz, "lam": hx(lam), "out": int(out), "first": fa.tolist()})
    with open(os.path.join(OUT, "status_traces.json"), "w") as f:
        json.dump(traces, f)

    # 4. KvStore LIFO block tables (kv_cache.cpp:53-55, 78-106, 182-194)
    kv = []
    for case, (L, pool, cap) in enumerate(((3, 48, 4), (8, 256, 16), (24, 4096, 16))):
        ops, caps, live = [], [], []
        nid, free, held = 0, pool, {}
        for _ in range(120):
            if rng.random() < 0.6 or not live:
                c = int(rng.integers(1, 40))
                need = -(-c // cap) * L
                ops.append(nid + 1); caps.append(c)
                if need <= free:  # otherwise KvOutOfMemory: the allocation is deferred (no table)
                    free -= need; held[nid] = need; live.append(nid)
                nid += 1
            else:
                i = int(rng.integers(len(live))); sid = live.pop(i)
                ops.append(-(sid + 1)); caps.append(0); free += held.pop(sid)
        bpl_max = 16
        tab, nf = R.kv_block_trace(L, pool, cap, ops, caps, nid, bpl_max)
        kv.append({"L": L, "pool": pool, "cap": cap, "ops": ops, "caps": caps, "n_ids": nid, "bpl_max": bpl_max,
                   "tables": tab.tolist(), "free": int(nf)})
    with open(os.path.join(OUT, "kv_block_traces.json"), "w") as f:
        json.dump(kv, f)

    # 5. gen_workload (workload.cpp:58-89)
    wls = []
    for p in ({"n_requests": 5, "mean_interarrival": 0.0, "prompt_len_min": 1, "prompt_len_max": 6,
               "output_len_min": 1, "output_len_max": 32, "seed": 500, "vocab_size": 256, "eos_token": 0},
              {"n_requests": 7, "mean_interarrival": 0.015, "prompt_len_min": 2, "prompt_len_max": 9,
               "output_len_min": 3, "output_len_max": 8, "seed": 11, "vocab_size": 32128, "eos_token": 0},
              {"n_requests": 4, "mean_interarrival": 0.0, "prompt_len_min": 512, "prompt_len_max": 512,
               "output_len_min": 128, "output_len_max": 128, "seed": 1, "vocab_size": 32128, "eos_token": 0}):
        w = R.gen_workload(**p)
        wls.append({"params": p, "arrival": hx(w.arrival), "prompt_off": w.prompt_off.tolist(),
                    "prompt": w.prompt.tolist(), "max_new": w.max_new.tolist()})
    with open(os.path.join(OUT, "workloads.json"), "w") as f:
        json.dump(wls, f)

    # 6. Engine::run transcripts on the acceptance corpus shape (acceptance.cpp:50-72)
    runs = []
    setups = [("never", {}), ("always_at", {"exit_layer": 4}), ("state", {"lambda0": 0.90}),
              ("softmax", {"lambda0": 0.02}), ("classifier", {"lambda0": 0.55})]
    for i in range(3):
        for tech, kw in setups:
            for rb in (False, True):
                cfg = B.engine_config(8, 64, 256, 1000 + i, tech, max_batch=8, pool_blocks=8192, round_bf16=rb, **kw)
                wl = R.gen_workload(n_requests=3 + i % 14, mean_interarrival=(i % 3) * 0.015, prompt_len_min=1,
                                    prompt_len_max=6, output_len_min=1, output_len_max=32, seed=500 + i,
                                    vocab_size=256)
                mm = R.model(8, 64, 256, 1000 + i, rb)
                t = mm.run(cfg, wl)
                rec = {"i": i, "tech": tech, "kw": kw, "round_bf16": rb}
                for fld in B.I32_FIELDS:
                    rec[fld] = t[fld].tolist()
                for fld in B.F64_FIELDS:
                    if fld != "it_conf":
                        rec[fld] = hx(t[fld])
                runs.append(rec)
    with open(os.path.join(OUT, "transcripts.json"), "w") as f:
        json.dump(runs, f)

    # 7. bench-workload decode (seeded KV prefix), restated over the reference's functions
    sess = []
    for tech, lam, gamma in (("state", 0.97, 0.995), ("softmax", 1e-7, 1.0), ("classifier", 0.55, 1.0)):
        cfg = B.engine_config(4, 128, 512, 5, tech, lambda0=lam, gamma=gamma, max_batch=8, pool_blocks=4096,
                              round_bf16=True, eos_token=-1)
        mm = R.model(4, 128, 512, 5, True)
        first = [3, 9, 27, 81, 243, 100]
        s = mm.session(cfg, first, 30, 48, 1234)
        steps = []
        for _ in range(3):
            o = s.step()
            steps.append({"e": int(o["output_layer"]), "tokens": o["tokens"].tolist(), "accept": o["accept"].tolist(),
                          "conf": hx(np.nan_to_num(o["conf"], nan=-7.0)), "h": hx(o["h_exit"][:, :8])})
        sess.append({"tech": tech, "lam": lam, "gamma": gamma, "first": first, "steps": steps})
    with open(os.path.join(OUT, "sessions.json"), "w") as f:
        json.dump(sess, f)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
