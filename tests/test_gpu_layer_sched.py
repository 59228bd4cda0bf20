"""f4: layer-level scheduling driving real batches (layer_sched.hpp's occupancy
MDP, whose policies the reference only simulates, layer_sched.hpp:18-19).

Each turn runs one layer for the sequences whose next layer it is; every sequence exits on its
own accept.  Per sequence this is exactly the reference's decode_iteration on a batch of one,
which the oracle runs as its per-sequence-exit session (pinned to single-sequence reference
sessions in tests/test_oracle_cpu.py).  The B200 sequences advance at different rates; each
row's token / exit-layer stream is compared with the oracle's stream for that row up to the
first near-tie divergence (a flipped decision within the confidence tolerance of lambda, or a
greedy token whose top-2 logit gap is below TIE_GAP), after which the inputs differ."""
import numpy as np
import pytest

import bench
from oracle import bindings as OB
from paper_2407_20272_b200 import exitlab as X

pytestmark = pytest.mark.gpu

CONF_TOL = {"state": 1e-4, "classifier": 1e-4}
TIE_GAP = 2e-2


def _run(port, L, d, V, B, tech, lam, gamma, turns, policy="greedy", M=None, prefix=40, defer=1):
    cfg = X.EngineConfig(model=X.ModelConfig(L, d, V, 0), technique=X.ExitTechnique(tech),
                         schedule=X.ThresholdSchedule(lam, gamma, 0.0), max_batch=B, pool_blocks=B * L * 16,
                         eos_token=-1)
    e = X.Engine(cfg)
    e.set_option("sched_defer", defer)  # deferred token turns (default) or a token per exiting row at once
    first = np.array([p[-1] % V for p in bench.workload(B)], np.int32)
    cap = prefix + 1 + 64
    e.session_begin(first, prefix, cap, 1, np.arange(B))
    e.sched_begin(policy, M)
    e.sched_run(turns)
    got = [e.sched_tokens(b) for b in range(B)]
    layers, rows = e.sched_turns()
    return e, first, got, layers, rows, cap


@pytest.mark.parametrize("L,d,V,B,tech,lam,gamma,defer", [(6, 256, 1024, 24, "state", 0.97, 0.998, 1),
                                                         (6, 256, 1024, 24, "state", 0.97, 0.998, 0),
                                                         (12, 768, 32128, 64, "state", 0.981, 0.997, 1),
                                                         (8, 512, 4096, 40, "classifier", 0.406, 0.999, 1)])
def test_layer_level_schedule_matches_single_sequence_decoding(port, L, d, V, B, tech, lam, gamma, defer):
    e, first, got, layers, rows, cap = _run(port, L, d, V, B, tech, lam, gamma, turns=8 * L, defer=defer)
    # every turn engages exactly the sequences at its layer (layer 0: a token turn)
    assert len(layers) == 8 * L and rows.min() >= 1
    assert (0 in set(layers.tolist())) == bool(defer)
    n_max = max(len(t) for t, _ in got)
    assert n_max >= 2 and sum(len(t) for t, _ in got) > B
    cfg = OB.engine_config(L, d, V, 0, tech, lambda0=lam, gamma=gamma, max_batch=B, pool_blocks=4096, eos_token=-1,
                           round_bf16=True)
    m = port.model(L, d, V, 0, True)
    s = m.session(cfg, first, 40, cap, 1, np.arange(B))
    s.set_per_seq_exit(True)
    lm = m.tensor("lm_head")
    lam_l = np.array([port.threshold_at(lam, gamma, 0.0, i) for i in range(1, L + 1)])
    div = [None] * B  # first oracle step where the row's input diverged
    agree_tok = agree_exit = total = 0
    exits_seen = set()
    tok_in = None
    for step in range(n_max):
        o = s.step(tokens_in=tok_in)
        tok_in = o["tokens"].copy()
        logits = o["h_exit"] @ lm.T
        top2 = np.sort(logits, axis=1)[:, -2:]
        for b in range(B):
            t, x = got[b]
            if div[b] is not None or step >= len(t):
                continue
            total += 1
            exits_seen.add(int(x[step]))
            same_exit = int(x[step]) == int(o["accept"][b])
            if not same_exit:  # a flipped decision: the oracle's confidence sits at lambda
                l = min(int(x[step]), int(o["accept"][b]))
                c = o["conf"][l - 1, b]
                assert abs(c - lam_l[l - 1]) <= CONF_TOL[tech], (b, step, l, c, lam_l[l - 1])
                div[b] = step
                continue
            agree_exit += 1
            if int(t[step]) != int(o["tokens"][b]):
                assert top2[b, 1] - top2[b, 0] < TIE_GAP, (b, step)
                div[b] = step
                continue
            agree_tok += 1
            tok_in[b] = t[step]  # keep the oracle on the B200's inputs
        # rows that diverged or ran out keep their own oracle inputs (not compared any more)
    print(dict(tokens_compared=total, exit_agree=agree_exit / total, token_agree=agree_tok / total,
               exit_layers_seen=sorted(exits_seen), turns=len(layers), mean_rows=float(rows.mean())))
    assert agree_exit / total >= 0.9 and agree_tok / total >= 0.9
    assert len(exits_seen) > 1  # sequences exit at their own layers
    e.close()


def test_linear_policy_identity_equals_greedy(port):
    """LinearQ::identity reproduces q_init = v[a] (layer_sched.hpp:92-95): the same schedule as
    greedy_action, turn for turn."""
    L, d, V, B = 6, 256, 1024, 24
    ea, _, ga, la, ra, _ = _run(port, L, d, V, B, "state", 0.97, 0.998, 30)
    eb, _, gb, lb, rb, _ = _run(port, L, d, V, B, "state", 0.97, 0.998, 30, policy="linear", M=np.eye(L))
    assert np.array_equal(la, lb) and np.array_equal(ra, rb)
    for (t1, x1), (t2, x2) in zip(ga, gb):
        assert np.array_equal(t1, t2) and np.array_equal(x1, x2)
    ea.close()
    eb.close()
