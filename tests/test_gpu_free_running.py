"""Free-running parity at the BASELINE configs (north_star: "greedy tokens and exit layers
agree at a reported rate, with near-threshold ties listed").

The oracle (the fp64 restatement of engine.cpp:208-310, bit-identical to the compiled
reference, on the same bf16-rounded weights) decodes the bench workload freely: its own exit
decisions, its own greedy tokens.  Each B200 decode strategy then runs the same iterations
with the oracle's input tokens (so every iteration starts from the same tokens) but takes its
OWN exit decisions -- nothing is forced.  Per iteration we compare:

* every exit decision (seq, layer) both engines evaluated (layers <= min of the two output
  layers): a decision may differ only where the oracle's confidence lies within the
  confidence tolerance of lambda_i (a near-threshold tie); every tie is listed;
* the output layer (iteration exit layer) and each sequence's accept layer -> agreement rates;
* the greedy tokens where both engines exited at the same layer: a disagreement must be a
  near-tie of the oracle's logits (top-2 gap < TIE_GAP) -> agreement rate;
* hidden states at the exit layer (same exit) and the K/V of the last position.

Reports go to $EL_PARITY_DIR (default gpurun_out/parity) as JSON; profiles/parity_r02.json
holds the committed copy.  Configs = bench.CONFIGS (calibrated thresholds).
"""
import json
import os

import numpy as np
import pytest

import bench
from oracle import bindings as OB
from paper_2407_20272_b200 import exitlab as X

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

V = 32128
# tolerances (bf16 weights and GEMM operands, fp32 accumulation / residual stream, against fp64)
CONF_TOL = {"state": 1e-4, "classifier": 1e-4}  # absolute (observed max 3.3e-5 over C2-C5, 16 iterations)
# softmax response p1 - p2 = (1 - exp(-(l1 - l2))) / sum exp(l - l1) ~ (l1 - l2) / V at V = 32128 with
# near-equal logits: bf16 hidden states move the top-2 logit gap by ~1e-4..3e-4 logit units, i.e.
# ~5e-9 in the confidence (observed max 4.7e-9 at C1, 8.6e-9 at C4 dims, 16 iterations) -> an
# absolute tolerance; at these dims the criterion itself sits below bf16 resolution
SM_ATOL = 1.5e-8
HID_TOL = 5e-3  # max|diff| / max|ref| of the exit hidden state when both engines exit at the same layer
KV_TOL = 8e-3   # the same for K/V rows (computed: vs the oracle; filled: vs fp64 W_kv h_e of the B200's h_e)
TIE_GAP = 2e-2  # oracle top-2 logit gap below which a greedy-token disagreement is a tie
ITERS = 16

CASES = [  # (bench config, decode strategy: True persistent kernel, False per-phase kernels)
    ("c1", False), ("c1", True),
    ("c2", True), ("c2", False),
    ("c3", True),
    ("c5", True),
    ("c4s", True),
    ("c4m", False), ("c4m", True),
]


def report_dir():
    d = os.environ.get("EL_PARITY_DIR", os.path.join(bench.ROOT, "gpurun_out", "parity"))
    os.makedirs(d, exist_ok=True)
    return d


_ORACLE = {}


def oracle_run(port, name):
    """The oracle's free-running trajectory of the bench workload (cached per config)."""
    if name in _ORACLE:
        return _ORACLE[name]
    c = bench.CONFIGS[name]
    L, d, B = c["L"], c["d"], c["B"]
    m = port.model(L, d, V, 0, True)
    cfg = OB.engine_config(L, d, V, 0, c["tech"], lambda0=c["lam"], gamma=c["gamma"], max_batch=B,
                           pool_blocks=4096, eos_token=-1, round_bf16=True)
    prompts = bench.workload(B)
    first = np.array([p[-1] for p in prompts], np.int32)
    s = m.session(cfg, first, bench.PROMPT - 1, bench.PROMPT + bench.OUT_LEN, 1, np.arange(B))
    lm = m.tensor("lm_head")
    recs, tin = [], first
    for _ in range(ITERS):
        o = s.step()
        logits = o["h_exit"] @ lm.T
        top2 = np.sort(logits, axis=1)[:, -2:]
        recs.append(dict(tin=tin.copy(), e=o["output_layer"], acc=o["accept"].copy(), conf=o["conf"].copy(),
                         h=o["h_exit"].copy(), tok=o["tokens"].copy(), gap=top2[:, 1] - top2[:, 0]))
        tin = o["tokens"].astype(np.int32)
    lam = np.array([port.threshold_at(c["lam"], c["gamma"], 0.0, l) for l in range(1, L + 1)])
    out = dict(recs=recs, first=first, lam=lam, model=m, session=s)
    _ORACLE.clear()  # one config's KV store at a time (C5: ~13 GB of host memory)
    _ORACLE[name] = out
    return out


def conf_tol(tech, conf_o):
    return np.full_like(conf_o, SM_ATOL if tech == "softmax" else CONF_TOL[tech])


@pytest.mark.parametrize("name,mega", CASES)
def test_free_running_parity(port, name, mega):
    c = bench.CONFIGS[name]
    L, d, B, tech = c["L"], c["d"], c["B"], c["tech"]
    orc = oracle_run(port, name)
    lam = orc["lam"]
    cfg = X.EngineConfig(model=X.ModelConfig(L, d, V, 0), technique=X.ExitTechnique(tech),
                         schedule=X.ThresholdSchedule(c["lam"], c["gamma"], 0.0), max_batch=B,
                         pool_blocks=B * L * 40, eos_token=-1)
    e = X.Engine(cfg, mega=mega)
    e.session_begin(orc["first"], bench.PROMPT - 1, bench.PROMPT + bench.OUT_LEN, 1, np.arange(B))
    ties, flips, rows = [], [], []
    max_conf_err = max_conf_rel = max_h = 0.0
    tok_same = tok_n = 0
    tok_untied_bad = []
    for i, o in enumerate(orc["recs"]):
        r = e.decode_iteration(o["tin"])
        eg, eo = int(r["output_layer"]), int(o["e"])
        n = min(eg, eo)
        cg, co = r["conf"][:n].astype(np.float64), o["conf"][:n]
        tol = conf_tol(tech, co)
        err = np.abs(cg - co)
        max_conf_err = max(max_conf_err, float(err.max()))
        max_conf_rel = max(max_conf_rel, float((err / np.maximum(np.abs(co), 1e-300)).max()))
        near = np.abs(co - lam[:n, None]) <= tol
        dg, do = cg > lam[:n, None], co > lam[:n, None]
        for l, b in zip(*np.nonzero(near)):
            ties.append(dict(iter=i, seq=int(b), layer=int(l) + 1, conf_oracle=float(co[l, b]),
                             conf_b200=float(cg[l, b]), lam=float(lam[l]), flipped=bool(dg[l, b] != do[l, b])))
        for l, b in zip(*np.nonzero(dg != do)):
            flips.append(dict(iter=i, seq=int(b), layer=int(l) + 1, conf_oracle=float(co[l, b]),
                              conf_b200=float(cg[l, b]), lam=float(lam[l]), tie=bool(near[l, b])))
        row = dict(iter=i, e_oracle=eo, e_b200=eg, accept_agree=float(np.mean(r["accept"] == o["acc"])))
        if eg == eo:
            h = e.hidden(eg & 1)
            hr = float(np.abs(h - o["h"]).max() / np.abs(o["h"]).max())
            max_h = max(max_h, hr)
            same = r["tokens"] == o["tok"]
            tok_same += int(same.sum())
            tok_n += B
            bad = ~same & (o["gap"] >= TIE_GAP)
            tok_untied_bad += [dict(iter=i, seq=int(b), gap=float(o["gap"][b])) for b in np.nonzero(bad)[0]]
            row.update(h_relerr=hr, token_agree=float(same.mean()))
        rows.append(row)
    # K/V of the last position vs the oracle (computed layers <= both exits) and vs the fp64
    # projection of the B200's own exit state (filled layers)
    last = orc["recs"][-1]
    pos = bench.PROMPT - 1 + ITERS - 1
    eg = rows[-1]["e_b200"]
    kv_err = fill_err = 0.0
    h_last = e.hidden(eg & 1).astype(np.float64)
    for b in (0, B - 1):
        for layer in range(1, L + 1):
            kg, vg = e.kv(b, layer, pos)
            if layer <= min(eg, last["e"]):
                ko, vo = orc["session"].kv(b, layer, pos)
                kv_err = max(kv_err, float(np.abs(kg - ko).max() / np.abs(ko).max()),
                             float(np.abs(vg - vo).max() / np.abs(vo).max()))
            elif layer > eg:
                kp = orc["model"].tensor("w_k", layer) @ h_last[b]
                vp = orc["model"].tensor("w_v", layer) @ h_last[b]
                fill_err = max(fill_err, float(np.abs(kg - kp).max() / np.abs(kp).max()),
                               float(np.abs(vg - vp).max() / np.abs(vp).max()))
    # the single-launch strategy runs the pipelined kernel at batch 65-256 (el_pipe.cuh)
    kernel = "per-phase" if not mega else ("pipelined" if e.plan_info().get("pipe") else "persistent")
    e.close()
    eo_all = np.array([x["e_oracle"] for x in rows])
    eg_all = np.array([x["e_b200"] for x in rows])
    summary = dict(config=name, workload=c["name"], strategy="persistent" if mega else "per-phase", kernel=kernel, technique=tech,
                   schedule=[c["lam"], c["gamma"]], batch=B, iterations=ITERS,
                   exit_layer_agreement=float(np.mean(eo_all == eg_all)),
                   accept_layer_agreement=float(np.mean([x["accept_agree"] for x in rows])),
                   token_agreement_same_exit=(tok_same / tok_n) if tok_n else None,
                   mean_exit_oracle=float(eo_all.mean()), mean_exit_b200=float(eg_all.mean()),
                   max_conf_abs_err=max_conf_err, max_conf_rel_err=max_conf_rel, max_h_relerr=max_h,
                   kv_relerr_last_pos=kv_err, fill_relerr_last_pos=fill_err,
                   n_near_threshold=len(ties), n_flipped=len(flips),
                   tolerances=dict(conf=SM_ATOL if tech == "softmax" else CONF_TOL[tech], h=HID_TOL, kv=KV_TOL,
                                   tie_gap=TIE_GAP),
                   iterations_detail=rows, near_threshold_ties=ties[:200], flipped=flips[:200],
                   token_disagreements_not_ties=tok_untied_bad[:50])
    with open(os.path.join(report_dir(), f"{name}_{summary['strategy']}.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({k: v for k, v in summary.items() if not isinstance(v, list)}))
    # every flipped decision is a near-threshold tie (and so every exit-layer disagreement)
    assert all(f["tie"] for f in flips), flips[:5]
    assert max_h <= HID_TOL, max_h
    assert not tok_untied_bad, tok_untied_bad[:5]
    assert kv_err <= KV_TOL and fill_err <= KV_TOL, (kv_err, fill_err)
