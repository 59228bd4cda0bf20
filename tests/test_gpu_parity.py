"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (north_star / SURVEY 8c):
* bit-exact: seeded bf16 weights, block tables, exit masks / first-accept /
  output layer at injected confidences, control plane of Engine::run
  (batch composition, clocks, charges, finish order) where exits are fixed.
* tolerance (bf16 weights AND activations entering the tensor cores, fp32
  residual stream / accumulation, oracle = fp64 reference on the same
  bf16-rounded weights, teacher-forced on the GPU's inputs and exit layer):
    hidden states / computed K,V      max|diff| / max|ref| <= HID_TOL
    filled K,V vs fp64 W_kv h_e       max|diff| / max|ref| <= FILL_TOL
    cos / classifier confidences      |diff| <= CONF_TOL
    softmax-response confidence       |diff| <= 0.01 * 4/V
    greedy tokens                     >= 90 % agree; every disagreement is a near-tie
                                      (oracle top-2 logit gap < TIE_GAP)
"""
import numpy as np
import pytest

from oracle import bindings as OB
from paper_2407_20272_b200 import exitlab as X

pytestmark = pytest.mark.gpu

HID_TOL = 3e-2
FILL_TOL = 2e-2
CONF_TOL = 3e-3
TIE_GAP = 2e-2


def cfg_pair(L, d, V, seed, tech="never", lam=0.85, gamma=1.0, exit_layer=1, B=8, pool=None, bc=16, eos=-1):
    pool = pool or B * L * 64
    g = X.EngineConfig(model=X.ModelConfig(L, d, V, seed), technique=X.ExitTechnique(tech, exit_layer),
                       schedule=X.ThresholdSchedule(lam, gamma, 0.0), max_batch=B, pool_blocks=pool,
                       block_capacity=bc, eos_token=eos)
    o = OB.engine_config(L, d, V, seed, tech, exit_layer=exit_layer, lambda0=lam, gamma=gamma, max_batch=B,
                         pool_blocks=pool, block_capacity=bc, eos_token=eos, round_bf16=True)
    return g, o


def relerr(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.fixture(scope="module")
def tiny():
    g, o = cfg_pair(3, 8, 16, 11, B=4, pool=256, bc=4)
    return g, o


def test_weights_bit_exact(port):
    for (L, d, V, seed) in ((3, 8, 16, 11), (2, 512, 32128, 0)):
        g, _ = cfg_pair(L, d, V, seed, B=2)
        e = X.Engine(g)
        m = port.model(L, d, V, seed, round_bf16=True)
        for name in ["embedding", "lm_head", "probe_w", "probe_b"]:
            assert np.array_equal(X.bf16_to_f64(e.model_tensor(name)).ravel(), m.tensor(name).ravel()), name
        for layer in range(1, L + 1):
            for name in ["w_q", "w_k", "w_v", "w_o", "w_up", "w_down"]:
                assert np.array_equal(X.bf16_to_f64(e.model_tensor(name, layer)), m.tensor(name, layer)), name
        e.close()


def test_never_equals_reference_decoder(port, tiny):
    # test_engine.cpp:98-109 on the device: technique never == reference_decode
    g, o = tiny
    e = X.Engine(g)
    m = port.model(3, 8, 16, 11, round_bf16=True)
    t = e.run(X.Workload([X.Request(0.0, [1, 2, 3], 6)]))
    assert t.sequences[0]["tokens"] == m.reference_decode([1, 2, 3], 6, 0)
    assert all(it["output_layer"] == 3 for it in t.iterations)


@pytest.mark.parametrize("graph", [True, False])
def test_engine_run_control_plane_bit_exact(port, graph):
    """FIFO admission, head-of-line deferral, eviction, clocks, charges and
    output layers (always_at) identical to the oracle (test_engine.cpp:153-205)."""
    for tech, kw in (("always_at", dict(exit_layer=2)), ("never", {})):
        g, o = cfg_pair(3, 8, 16, 11, tech, B=4, pool=12, bc=4, eos=-1, **kw)
        e = X.Engine(g, graph=graph)
        reqs = [(0.0, [1, 2, 3, 4], 8), (0.0, [5, 6, 7, 8], 12), (0.0, [9], 1), (0.02, [3, 3], 3)]
        t = e.run(X.Workload([X.Request(*r) for r in reqs]))
        wl = OB.Workload.from_requests(reqs)
        tp = port.model(3, 8, 16, 11, True).run(o, wl)
        for f in ["it_output_layer", "it_batch_off", "ps_seq", "ps_accept", "sq_id", "sq_max_new", "pf_seq",
                  "pf_positions", "sq_iter_out", "sq_exit_layers"]:
            assert np.array_equal(t[f], tp[f]), (tech, f)
        for f in ["it_clock", "it_charge", "pf_clock", "sq_arrival", "sq_first", "sq_finish", "meta"]:
            assert np.array_equal(t[f], tp[f]), (tech, f)
        # deferral: id 1 (12 blocks) waits; id 2 is blocked behind it (strict FIFO)
        first = {}
        for i, it in enumerate(t.iterations):
            for sid in it["batch_ids"]:
                first.setdefault(sid, i)
        assert first[0] == 0 and first[1] > first[0] and first[2] > first[1]
        e.close()


def test_block_tables_bit_exact(port):
    L, B, cap, bc = 4, 6, 50, 16
    g, o = cfg_pair(L, 128, 512, 3, B=B, pool=B * L * 4 + 5, bc=bc)
    e = X.Engine(g)
    e.session_begin(np.arange(B) + 1, 20, cap, 9)
    bpl = -(-cap // bc)
    ops = list(range(1, B + 1))
    want, _ = port.kv_block_trace(L, g.pool_blocks, bc, ops, [cap] * B, B, bpl)
    host, _ = X.kv_block_trace(L, g.pool_blocks, bc, ops, [cap] * B, B, bpl)
    for b in range(B):
        got = e.block_table(b)
        assert np.array_equal(got, want[b]) and np.array_equal(host[b], want[b])
    e.close()


@pytest.mark.parametrize("graph,mega", [(True, False), (False, False), (True, True)])
def test_exit_masks_bit_exact_at_fixed_confidences(port, graph, mega):
    """ExitStatusVector on the device == reference semantics at injected
    confidences: OR-latch, first accept, output layer = max accept, strict '>'."""
    L, B = 6, 12
    g, o = cfg_pair(L, 128, 512, 3, "fixed", lam=0.6, gamma=0.97, B=B)
    e = X.Engine(g, graph=graph, mega=mega)
    e.session_begin(np.arange(B) + 5, 8, 8 + 40, 2)
    rng = np.random.default_rng(0)
    lam = np.array([OB.port().threshold_at(0.6, 0.97, 0.0, l) for l in range(1, L + 1)])
    for it in range(30):
        conf = rng.random((L, B)).astype(np.float32)
        if it % 5 == 0:
            conf[:] = 0.0  # nobody exits -> output layer L
        if it % 7 == 3:
            conf[2, :] = np.float32(1.0)  # everybody at layer 3
        # exact ties: conf == lambda must reject (strict >)
        conf[0, 0] = np.float32(lam[0])
        e.set_fixed_confidences(conf)
        r = e.decode_iteration()
        # the device compares (double)float(conf) > lambda: feed the same float values to the oracle
        want_e, want_fa = port.status_trace(conf.astype(np.float64), lam)
        assert r["output_layer"] == want_e, it
        assert r["accept"].tolist() == want_fa.tolist(), it
    e.close()


def _teacher_forced(e, s, n_iters, lm, V, d, check_conf=None):
    """Run n iterations on the GPU; replay each on the oracle with the GPU's
    input tokens and exit layer; return per-iteration error stats."""
    stats = []
    tok_in = None
    for _ in range(n_iters):
        r = e.decode_iteration()
        ex = r["output_layer"]
        o = s.step(forced=ex, tokens_in=tok_in)
        h_gpu = e.hidden(ex & 1)
        logits = o["h_exit"] @ lm.T
        top2 = np.sort(logits, axis=1)[:, -2:]
        gap = top2[:, 1] - top2[:, 0]
        agree = r["tokens"] == o["tokens"]
        conf_err = 0.0
        for l in range(ex):
            cg, co = r["conf"][l].astype(np.float64), o["conf"][l]
            m = ~np.isnan(co)
            if m.any():
                conf_err = max(conf_err, float(np.abs(cg[m] - co[m]).max()))
        stats.append(dict(e=ex, h=relerr(h_gpu, o["h_exit"]), agree=agree, gap=gap, conf=conf_err,
                          tokens=r["tokens"].copy(), h_exit=h_gpu, h_oracle=o["h_exit"]))
        tok_in = r["tokens"]  # next iteration: the oracle consumes the GPU's tokens
    return stats


@pytest.mark.parametrize("mega", [False, True])
@pytest.mark.parametrize("tech,lam,gamma", [("state", 0.972, 0.998), ("classifier", 0.59, 1.0),
                                            ("softmax", 1e-4, 1.0), ("always_at", 0.5, 1.0), ("never", 0.5, 1.0)])
def test_decode_parity_small_dims(port, tech, lam, gamma, mega):
    """Both decode strategies (per-phase kernels; persistent kernel) against the oracle."""
    L, d, V, B = 4, 128, 512, 8
    g, o = cfg_pair(L, d, V, 5, tech, lam=lam, gamma=gamma, exit_layer=2, B=B)
    e = X.Engine(g, mega=mega)
    first = np.array([3, 9, 27, 81, 243, 100, 7, 500])
    e.session_begin(first, 30, 60, 1234)
    m = port.model(L, d, V, 5, True)
    s = m.session(o, first, 30, 60, 1234)
    st = _teacher_forced(e, s, 6, m.tensor("lm_head"), V, d)
    tol_sm = 0.01 * 4.0 / V
    for x in st:
        assert x["h"] <= HID_TOL, x["h"]
        assert x["conf"] <= (tol_sm if tech == "softmax" else CONF_TOL), x["conf"]
        assert np.all(x["agree"] | (x["gap"] < TIE_GAP)), x["gap"][~x["agree"]]
    agree = np.mean([x["agree"].mean() for x in st])
    assert agree >= 0.9
    if tech == "always_at":
        assert all(x["e"] == 2 for x in st)
    if tech == "never":
        assert all(x["e"] == L for x in st)
    # KV of the last position: computed layers vs oracle, filled layers vs fp64 projection of h_e
    pos = 30 + len(st) - 1
    ex = st[-1]["e"]
    for layer in range(1, L + 1):
        kg, vg = e.kv(0, layer, pos)
        ko, vo = s.kv(0, layer, pos)
        assert relerr(kg, ko) <= HID_TOL and relerr(vg, vo) <= HID_TOL, layer
        if layer > ex:
            h = st[-1]["h_exit"][0].astype(np.float64)
            kp = m.tensor("w_k", layer) @ h
            vp = m.tensor("w_v", layer) @ h
            assert relerr(kg, kp) <= FILL_TOL and relerr(vg, vp) <= FILL_TOL, layer
    e.close()


def test_graph_equals_eager_bitwise():
    L, d, V, B = 6, 256, 1024, 16
    outs = []
    for graph in (True, False):
        g, _ = cfg_pair(L, d, V, 8, "state", lam=0.97, gamma=0.995, B=B)
        e = X.Engine(g, graph=graph)
        e.session_begin(np.arange(B) * 3 + 1, 40, 80, 77)
        rs = [e.decode_iteration() for _ in range(5)]
        outs.append((rs, e.hidden(rs[-1]["output_layer"] & 1), e.kv(3, L, 44)))
        e.close()
    (ra, ha, ka), (rb, hb, kb) = outs
    for x, y in zip(ra, rb):
        assert x["output_layer"] == y["output_layer"]
        assert np.array_equal(x["tokens"], y["tokens"]) and np.array_equal(x["conf"], y["conf"])
    assert np.array_equal(ha, hb) and np.array_equal(ka[0], kb[0])


def test_device_resident_run_matches_stepwise():
    L, d, V, B = 6, 256, 1024, 16
    res = []
    for mode in ("step", "run"):
        g, _ = cfg_pair(L, d, V, 8, "classifier", lam=0.55, B=B)
        e = X.Engine(g)
        e.session_begin(np.arange(B) * 5 + 2, 40, 80, 7)
        if mode == "step":
            toks = [e.decode_iteration()["tokens"] for _ in range(6)]
        else:
            e.decode_run(6)
            toks = list(e.records(0, 6)["tokens"])
        res.append(np.array(toks))
        e.close()
    assert np.array_equal(res[0], res[1])


def test_engine_run_with_real_prefill_matches_oracle(port):
    """Engine::run end to end (real prefill, ragged prompts, EOS): control plane
    bit-exact and tokens agreeing for the never technique (acceptance C1 shape)."""
    L, d, V = 4, 64, 256
    g, o = cfg_pair(L, d, V, 1000, "never", B=8, pool=8192, eos=0)
    e = X.Engine(g)
    wl = port.gen_workload(n_requests=6, mean_interarrival=0.0, prompt_len_min=1, prompt_len_max=6, output_len_min=1,
                           output_len_max=12, seed=500, vocab_size=V)
    t = e.run(X.Workload.from_flat(wl.arrival, wl.prompt_off, wl.prompt, wl.max_new))
    tp = port.model(L, d, V, 1000, True).run(o, wl)
    gt = {s["id"]: s["tokens"] for s in t.sequences}
    pt = {s["id"]: s["tokens"] for s in tp.sequences}
    agree = [a == b for k in pt for a, b in zip(gt[k], pt[k])]
    assert np.mean(agree) >= 0.9
    # reference_decode per sequence on the same weights
    m = port.model(L, d, V, 1000, True)
    for s in tp.sequences:
        assert m.reference_decode(s["prompt"], s["max_new"], 0) == s["tokens"]
    e.close()


@pytest.mark.slow
@pytest.mark.parametrize("mega", [False, True])
def test_bench_config_c2_parity(port, mega):
    """BASELINE configs[1] dims (L=12, d=768, V=32128), B=64, state exit: the
    bench workload itself, two teacher-forced iterations, both decode strategies."""
    L, d, V, B = 12, 768, 32128, 64
    g, o = cfg_pair(L, d, V, 0, "state", lam=0.972, gamma=0.998, B=B)
    e = X.Engine(g, mega=mega)
    wl = port.gen_workload(n_requests=B, prompt_len_min=512, prompt_len_max=512, output_len_min=128,
                           output_len_max=128, seed=1, vocab_size=V)
    first = wl.prompt[wl.prompt_off[1:] - 1]
    e.session_begin(first, 511, 640, 1)
    m = port.model(L, d, V, 0, True)
    s = m.session(o, first, 511, 640, 1)
    st = _teacher_forced(e, s, 2, m.tensor("lm_head"), V, d)
    for x in st:
        assert x["h"] <= HID_TOL and x["conf"] <= CONF_TOL
        assert np.all(x["agree"] | (x["gap"] < TIE_GAP))
    e.close()


@pytest.mark.parametrize("B,tech", [(16, "classifier"), (136, "state"), (256, "classifier")])
def test_persistent_kernel_deterministic_and_matches_per_phase(B, tech):
    """The persistent kernel is run-to-run bitwise deterministic (fixed split-K
    and attention-partial reduction orders, no atomics on values) and agrees
    with the per-phase kernels within the bf16 tolerance; B = 136 exercises the
    split-K + reduce GEMM path (activation rows not a multiple of 128), B = 16
    the batch-M path, B = 256 batch-M over two 128-row groups."""
    L, d, V = 5, 256, 1024
    outs = []
    for mega in (True, True, False):
        g, _ = cfg_pair(L, d, V, 8, tech, lam=0.97 if tech == "state" else 0.5, gamma=0.995, B=B)
        e = X.Engine(g, mega=mega)
        e.session_begin(np.arange(B) * 3 + 1, 40, 80, 77)
        rs = [e.decode_iteration() for _ in range(4)]
        outs.append((rs, e.hidden(rs[-1]["output_layer"] & 1), e.kv(B - 1, L, 43)))
        e.close()
    (ra, ha, ka), (rb, hb, kb), (rc, hc, kc) = outs
    for x, y in zip(ra, rb):
        assert x["output_layer"] == y["output_layer"]
        assert np.array_equal(x["tokens"], y["tokens"]) and np.array_equal(x["conf"], y["conf"])
    assert np.array_equal(ha, hb) and np.array_equal(ka[0], kb[0]) and np.array_equal(ka[1], kb[1])
    assert relerr(ha, hc) <= HID_TOL and relerr(ka[0], kc[0]) <= HID_TOL
    assert np.mean([np.mean(x["tokens"] == y["tokens"]) for x, y in zip(ra, rc)]) >= 0.9


@pytest.mark.parametrize("B", [8, 136])
@pytest.mark.parametrize("tech,lam,gamma", [("state", 0.972, 0.998), ("classifier", 0.59, 1.0), ("never", 0.5, 1.0)])
def test_t5_cross_attention_parity(port, tech, lam, gamma, B):
    """T5 mode (north_star (1): cross-attention over encoder states; no reference
    counterpart -- oracle = the C restatement, itself checked against an independent
    numpy decoder in test_t5_oracle_cpu.py).  B = 8 runs the batch-M GEMM phases,
    B = 136 the split-K + reduce phases of the persistent kernel."""
    L, d, V, T = 4, 128, 512, 24
    g = X.EngineConfig(model=X.ModelConfig(L, d, V, 5, encoder_len=T), technique=X.ExitTechnique(tech, 2),
                       schedule=X.ThresholdSchedule(lam, gamma, 0.0), max_batch=B, pool_blocks=B * L * 8,
                       eos_token=-1)
    o = OB.engine_config(L, d, V, 5, tech, exit_layer=2, lambda0=lam, gamma=gamma, max_batch=B,
                         pool_blocks=B * L * 8, eos_token=-1, round_bf16=True)
    e = X.Engine(g)
    first = (np.arange(B) * 37 + 3) % V
    e.session_begin(first, 30, 60, 1234)
    m = port.model(L, d, V, 5, True, encoder_len=T)
    s = m.session(o, first, 30, 60, 1234)
    st = _teacher_forced(e, s, 3, m.tensor("lm_head"), V, d)
    for x in st:
        assert x["h"] <= HID_TOL, x["h"]
        assert x["conf"] <= CONF_TOL, x["conf"]
        assert np.all(x["agree"] | (x["gap"] < TIE_GAP)), x["gap"][~x["agree"]]
    assert np.mean([x["agree"].mean() for x in st]) >= 0.9
    pos = 30 + len(st) - 1
    for layer in range(1, L + 1):
        kg, vg = e.kv(1, layer, pos)
        ko, vo = s.kv(1, layer, pos)
        assert relerr(kg, ko) <= HID_TOL and relerr(vg, vo) <= HID_TOL, layer
    e.close()


@pytest.mark.parametrize("L,d,heads,B,T", [(4, 128, 4, 8, 24), (3, 128, 16, 136, 40), (3, 512, 8, 16, 48),
                                           (2, 1024, 16, 64, 32), (3, 256, 4, 24, 0)])
def test_multi_head_parity(port, L, d, heads, B, T):
    """Attention split into heads (extension; head_dim 32 / 8 / 64 / 64 / 64: 4 / 1 / 8 / 8 / 8 lanes
    per head and chunk group; batch-M and split-K phases; T5 mode, and decoder-only with T = 0) vs
    the oracle's per-head restatement (pinned to an independent numpy decoder,
    tests/test_t5_oracle_cpu.py)."""
    V = 512
    g = X.EngineConfig(model=X.ModelConfig(L, d, V, 5, encoder_len=T, n_heads=heads),
                       technique=X.ExitTechnique("state"), schedule=X.ThresholdSchedule(0.972, 0.998, 0.0),
                       max_batch=B, pool_blocks=B * L * 8, eos_token=-1)
    o = OB.engine_config(L, d, V, 5, "state", lambda0=0.972, gamma=0.998, max_batch=B, pool_blocks=B * L * 8,
                         eos_token=-1, round_bf16=True)
    e = X.Engine(g)
    first = (np.arange(B) * 37 + 3) % V
    e.session_begin(first, 30, 60, 1234)
    m = port.model(L, d, V, 5, True, encoder_len=T, n_heads=heads)
    s = m.session(o, first, 30, 60, 1234)
    st = _teacher_forced(e, s, 3, m.tensor("lm_head"), V, d)
    for x in st:
        assert x["h"] <= HID_TOL, x["h"]
        assert x["conf"] <= CONF_TOL, x["conf"]
        assert np.all(x["agree"] | (x["gap"] < TIE_GAP)), x["gap"][~x["agree"]]
    assert np.mean([x["agree"].mean() for x in st]) >= 0.9
    # (random-init attention is near-uniform, so this only shows the split does no harm; the
    #  per-head softmax itself is checked with sharp attention in test_gpu_subengine.py)
    e.close()


@pytest.mark.parametrize("L,d,heads,B,T,NE", [(3, 128, 1, 8, 24, 2), (2, 256, 4, 12, 64, 3), (2, 1024, 8, 3, 256, 2)])
def test_t5_encoder_stack_parity(port, L, d, heads, B, T, NE):
    """T5 mode with a real encoder stack (NE bidirectional layers over seeded encoder ids, run at
    admission on the persistent kernel, 256 / T sequences per launch) feeding the cross K/V, vs the
    oracle's encoder restatement (pinned to an independent numpy encoder, test_t5_oracle_cpu.py)."""
    V = 512
    g = X.EngineConfig(model=X.ModelConfig(L, d, V, 5, encoder_len=T, n_heads=heads, encoder_layers=NE),
                       technique=X.ExitTechnique("state"), schedule=X.ThresholdSchedule(0.972, 0.998, 0.0),
                       max_batch=B, pool_blocks=B * L * 8, eos_token=-1)
    o = OB.engine_config(L, d, V, 5, "state", lambda0=0.972, gamma=0.998, max_batch=B, pool_blocks=B * L * 8,
                         eos_token=-1, round_bf16=True)
    e = X.Engine(g)
    first = (np.arange(B) * 37 + 3) % V
    e.session_begin(first, 30, 60, 1234)
    m = port.model(L, d, V, 5, True, encoder_len=T, n_heads=heads, encoder_layers=NE)
    s = m.session(o, first, 30, 60, 1234)
    st = _teacher_forced(e, s, 3, m.tensor("lm_head"), V, d)
    for x in st:
        assert x["h"] <= HID_TOL, x["h"]
        assert x["conf"] <= CONF_TOL, x["conf"]
        assert np.all(x["agree"] | (x["gap"] < TIE_GAP)), x["gap"][~x["agree"]]
    assert np.mean([x["agree"].mean() for x in st]) >= 0.9
    # the cross K/V of layer 1 come from the encoder output: compare them with the oracle's
    # W_kc / W_vc applied to its encoder states (bf16 storage)
    wkc, wvc = m.tensor("w_kc", 1), m.tensor("w_vc", 1)
    E = np.stack([m.encoder_state(1, t) for t in range(T)])
    kc, vc = e.cross_kv(1, 1)
    assert relerr(kc[:T], E @ wkc.T) <= 1e-2 and relerr(vc[:T], E @ wvc.T) <= 1e-2
    e.close()


def test_multi_head_config_checks():
    for heads, enc in ((3, 16), (64, 16), (32, 0)):  # no divisor; > 32 heads; head_dim 4 < 8
        with pytest.raises(ValueError):
            X.Engine(X.EngineConfig(model=X.ModelConfig(2, 128, 64, 1, encoder_len=enc, n_heads=heads),
                                    technique=X.ExitTechnique("never"), max_batch=2, pool_blocks=64))


@pytest.mark.parametrize("NE", [0, 2])
def test_t5_engine_run_matches_oracle(port, NE):
    """Engine::run in T5 mode (decoder prompt = start token, input in the encoder; NE > 0: the
    encoder stack runs at each admission)."""
    L, d, V, T = 3, 64, 256, 16
    g = X.EngineConfig(model=X.ModelConfig(L, d, V, 9, encoder_len=T, encoder_layers=NE),
                       technique=X.ExitTechnique("never"), max_batch=4, pool_blocks=512, eos_token=-1)
    o = OB.engine_config(L, d, V, 9, "never", max_batch=4, pool_blocks=512, eos_token=-1, round_bf16=True)
    reqs = [(0.0, [1], 6), (0.0, [5], 4), (0.0, [9], 7), (0.01, [2], 3), (0.02, [7], 5)]
    e = X.Engine(g)
    t = e.run(X.Workload([X.Request(*r) for r in reqs]))
    tp = port.model(L, d, V, 9, True, encoder_len=T, encoder_layers=NE).run(o, OB.Workload.from_requests(reqs))
    for f in ["it_output_layer", "it_batch_off", "ps_seq", "sq_id"]:
        assert np.array_equal(t[f], tp[f]), f
    gt = {s["id"]: s["tokens"] for s in t.sequences}
    pt = {s["id"]: s["tokens"] for s in tp.sequences}
    assert np.mean([a == b for k in pt for a, b in zip(gt[k], pt[k])]) >= 0.9
    with pytest.raises(ValueError):  # decoder prompts are the start token in T5 mode
        e.run(X.Workload([X.Request(0.0, [1, 2], 2)]))
    e.close()


@pytest.mark.parametrize("mega", [False, True])
def test_batched_prefill_kv_matches_oracle(port, mega):
    """f1: the prompt's K/V of every layer after Engine::run's prefill (engine.cpp:166-181).
    mega=True runs the batched causal prefill on the persistent kernel (rows = prompt
    positions, several per sequence per launch, max_batch rows per launch); mega=False the
    per-position per-phase path.  Both vs the oracle's token-by-token fp64 prefill."""
    L, d, V, B = 3, 128, 512, 6
    g = X.EngineConfig(model=X.ModelConfig(L, d, V, 21), technique=X.ExitTechnique("never"), max_batch=B,
                       pool_blocks=4096, eos_token=-1, capture_kv=True)
    o = OB.engine_config(L, d, V, 21, "never", max_batch=B, pool_blocks=4096, eos_token=-1, capture_kv=True,
                         round_bf16=True)
    rng = np.random.default_rng(5)
    reqs = [(0.0, [int(x) for x in rng.integers(1, V, n)], 2) for n in (41, 7, 33, 1, 58, 20)]
    e = X.Engine(g, mega=mega)
    t = e.run(X.Workload([X.Request(*r) for r in reqs]))
    tp = port.model(L, d, V, 21, True).run(o, OB.Workload.from_requests(reqs))
    for sid in range(len(reqs)):
        for layer in range(1, L + 1):
            kg, vg = t.kv(sid, layer)
            ko, vo = port.transcript_kv(tp, sid, layer, d)
            n = len(reqs[sid][1]) - 1  # prefill positions
            if n == 0:
                continue
            assert relerr(kg[:n], ko[:n]) <= HID_TOL and relerr(vg[:n], vo[:n]) <= HID_TOL, (sid, layer)
    gt = {s["id"]: s["tokens"] for s in t.sequences}
    pt = {s["id"]: s["tokens"] for s in tp.sequences}
    assert np.mean([a == b for k in pt for a, b in zip(gt[k], pt[k])]) >= 0.9
    e.close()


def test_batched_prefill_and_pipelined_decode_at_batch_144(port):
    """f1 with more than 128 sequences (position-major prefill launches of up to 144 rows on the
    persistent kernel -- the pipelined kernel measured slower for prefill, whose short early
    contexts leave its attention CTAs idle) and the pipelined decode at batch 144, small dims.
    K/V of every layer and the tokens vs the oracle's token-by-token fp64 prefill."""
    L, d, V, B = 3, 128, 512, 144
    g = X.EngineConfig(model=X.ModelConfig(L, d, V, 23), technique=X.ExitTechnique("never"), max_batch=B,
                       pool_blocks=8192, eos_token=-1, capture_kv=True)
    o = OB.engine_config(L, d, V, 23, "never", max_batch=B, pool_blocks=8192, eos_token=-1, capture_kv=True,
                         round_bf16=True)
    rng = np.random.default_rng(9)
    reqs = [(0.0, [int(x) for x in rng.integers(1, V, 2 + (i * 7) % 9)], 2) for i in range(B)]
    e = X.Engine(g, mega=True)
    t = e.run(X.Workload([X.Request(*r) for r in reqs]))
    tp = port.model(L, d, V, 23, True).run(o, OB.Workload.from_requests(reqs))
    for sid in range(0, B, 7):
        n = len(reqs[sid][1]) - 1
        for layer in range(1, L + 1):
            kg, vg = t.kv(sid, layer)
            ko, vo = port.transcript_kv(tp, sid, layer, d)
            assert relerr(kg[:n], ko[:n]) <= HID_TOL and relerr(vg[:n], vo[:n]) <= HID_TOL, (sid, layer)
    gt = {s["id"]: s["tokens"] for s in t.sequences}
    pt = {s["id"]: s["tokens"] for s in tp.sequences}
    assert np.mean([a == b for k in pt for a, b in zip(gt[k], pt[k])]) >= 0.9
    e.close()


def test_transcript_jsonl_byte_identical_on_device(port, tmp_path):
    """f3: the B200 engine's transcript written in the reference's JSONL format is byte-identical
    to the oracle's (and so to the reference's writer, tests/test_transcript_jsonl_cpu.py) when
    the decisions are fixed (technique never / always_at, tiny model: tokens equal too)."""
    for tech, kw in (("never", {}), ("always_at", dict(exit_layer=2))):
        g, o = cfg_pair(3, 8, 16, 11, tech, B=4, pool=64, bc=4, eos=-1, **kw)
        reqs = [(0.0, [1, 2, 3], 5), (0.0, [4, 5], 3), (0.01, [6], 4)]
        e = X.Engine(g)
        t = e.run(X.Workload([X.Request(*r) for r in reqs]))
        tp = port.model(3, 8, 16, 11, True).run(o, OB.Workload.from_requests(reqs))
        a, b = tmp_path / f"gpu_{tech}.jsonl", tmp_path / f"port_{tech}.jsonl"
        t.to_jsonl(str(a))
        X.write_transcript_jsonl(tp, str(b), g.model, g.technique)
        assert a.read_bytes() == b.read_bytes(), tech
        e.close()


@pytest.mark.parametrize("B", [200, 256])
def test_pipelined_kernel_matches_persistent_kernel(B):
    """The pipelined iteration kernel (el_pipe.cuh: attention and projection GEMMs of the two
    batch halves overlapped on disjoint CTA sets) against the plain persistent kernel on the same
    session: identical exit decisions and tokens up to split-K summation order (the down
    projection's K splits differ), run-to-run bitwise deterministic; B = 200 has a ragged second
    half."""
    L, d, V = 6, 1024, 2048
    outs = []
    for pipe in (1, 1, 0):
        g, _ = cfg_pair(L, d, V, 8, "classifier", lam=0.6, gamma=0.97, B=B)
        e = X.Engine(g, mega=True)
        e.set_option("pipe", pipe)
        e.session_begin(np.arange(B) * 7 % V + 1, 60, 100, 5)
        rs = [e.decode_iteration() for _ in range(4)]
        outs.append((rs, e.hidden(rs[-1]["output_layer"] & 1), e.kv(B - 1, L, 63), e.kv(3, 1, 63)))
        e.close()
    (ra, ha, ka, qa), (rb, hb, kb, qb), (rc, hc, kc, qc) = outs
    for x, y in zip(ra, rb):
        assert x["output_layer"] == y["output_layer"] and np.array_equal(x["tokens"], y["tokens"])
    assert np.array_equal(ha, hb) and np.array_equal(ka[0], kb[0]) and np.array_equal(qa[1], qb[1])
    assert [x["output_layer"] for x in ra] == [x["output_layer"] for x in rc]
    assert np.mean([np.mean(x["tokens"] == y["tokens"]) for x, y in zip(ra, rc)]) >= 0.97
    assert relerr(qa[0], qc[0]) <= 1e-2  # layer-1 K of the last position: same inputs, same GEMM


@pytest.mark.parametrize("B,tech,lam", [(128, "classifier", 0.6), (100, "classifier", 0.6), (100, "softmax", 2.0),
                                        (128, "softmax", 2.0)])
def test_pipelined_kernel_64_row_halves_match_persistent_kernel(B, tech, lam):
    """The pipelined kernel at batch 65-128 (halves of 64 rows, UMMA M = 64 batch-M groups; B = 100
    has a ragged second half of 36 rows; softmax: the LM-head check on the GEMM CTAs, lam 2.0 keeps
    every check to full depth) against the persistent kernel on the same session (max_batch 128):
    same exit decisions, tokens up to summation order, run-to-run bitwise deterministic."""
    L, d, V = 6, 1024, 2048
    outs = []
    for pipe in (1, 1, 0):
        g, _ = cfg_pair(L, d, V, 8, tech, lam=lam, gamma=0.97, B=128)
        e = X.Engine(g, mega=True)
        e.set_option("pipe", pipe)
        e.session_begin(np.arange(B) * 7 % V + 1, 60, 100, 5)
        assert e.plan_info()["pipe"] == (1 if pipe else 0)
        rs = [e.decode_iteration() for _ in range(4)]
        outs.append((rs, e.hidden(rs[-1]["output_layer"] & 1), e.kv(B - 1, L, 63), e.kv(3, 1, 63)))
        e.close()
    (ra, ha, ka, qa), (rb, hb, kb, qb), (rc, hc, kc, qc) = outs
    for x, y in zip(ra, rb):
        assert x["output_layer"] == y["output_layer"] and np.array_equal(x["tokens"], y["tokens"])
    assert np.array_equal(ha, hb) and np.array_equal(ka[0], kb[0]) and np.array_equal(qa[1], qb[1])
    assert [x["output_layer"] for x in ra] == [x["output_layer"] for x in rc]
    assert np.mean([np.mean(x["tokens"] == y["tokens"]) for x, y in zip(ra, rc)]) >= 0.97
    assert relerr(ha[:B], hc[:B]) <= 1e-2
    assert relerr(qa[0], qc[0]) <= 1e-2 and relerr(ka[0], kc[0]) <= 1e-2


@pytest.mark.parametrize("B,tech,lam", [(64, "state", 0.9), (48, "classifier", 0.6)])
def test_pipelined_kernel_32_row_halves_match_persistent_kernel(B, tech, lam):
    """The pipelined kernel at batch 33-64 (option pipe64: halves of 32 rows, UMMA M = 64 over a
    32-row group with the upper accumulator rows discarded; B = 48 has a ragged second half)
    against the persistent kernel on the same session (max_batch 64)."""
    L, d, V = 6, 768, 2048
    outs = []
    for pipe in (1, 1, 0):
        g, _ = cfg_pair(L, d, V, 8, tech, lam=lam, gamma=0.97, B=64)
        e = X.Engine(g, mega=True)
        e.set_option("pipe64", 1)
        e.set_option("pipe", pipe)
        e.session_begin(np.arange(B) * 7 % V + 1, 60, 100, 5)
        assert e.plan_info()["pipe"] == (1 if pipe else 0)
        rs = [e.decode_iteration() for _ in range(4)]
        outs.append((rs, e.hidden(rs[-1]["output_layer"] & 1), e.kv(B - 1, L, 63), e.kv(3, 1, 63)))
        e.close()
    (ra, ha, ka, qa), (rb, hb, kb, qb), (rc, hc, kc, qc) = outs
    for x, y in zip(ra, rb):
        assert x["output_layer"] == y["output_layer"] and np.array_equal(x["tokens"], y["tokens"])
    assert np.array_equal(ha, hb) and np.array_equal(ka[0], kb[0]) and np.array_equal(qa[1], qb[1])
    assert [x["output_layer"] for x in ra] == [x["output_layer"] for x in rc]
    assert np.mean([np.mean(x["tokens"] == y["tokens"]) for x, y in zip(ra, rc)]) >= 0.97
    assert relerr(ha[:B], hc[:B]) <= 1e-2
    assert relerr(qa[0], qc[0]) <= 1e-2 and relerr(ka[0], kc[0]) <= 1e-2


@pytest.mark.parametrize("B", [128, 256])
def test_lm_head_unit_variants_agree(B):
    """The LM-head unit variants give the same decisions and tokens: the softmax check on single
    tiles / pair units with the shuffle epilogue / transposed pair units (lm_pair 0 / 1 / 2, the
    persistent kernel at full depth), and the decode tail's greedy head on single tiles or
    transposed units (lm_tail 0 / 1, classifier exit: persistent at 128, pipelined at 256)."""
    L, d, V = 4, 1024, 4096
    first = np.arange(B) * 13 % V + 1
    if B == 128:
        runs = []
        for k in (0, 1, 2):
            g, _ = cfg_pair(L, d, V, 3, "softmax", lam=2.0, B=B)
            e = X.Engine(g, mega=True)
            e.set_option("pipe", 0)
            e.set_option("lm_pair", k)
            e.session_begin(first, 60, 100, 5)
            e.decode_run(3)
            runs.append(e.records(0, 3))
            e.close()
        for r in runs[1:]:
            assert np.array_equal(r["output_layer"], runs[0]["output_layer"])
            assert np.array_equal(r["tokens"], runs[0]["tokens"])
            np.testing.assert_allclose(r["conf"], runs[0]["conf"], rtol=1e-4, atol=1e-12)
    runs = []
    for k in (0, 1):
        g, _ = cfg_pair(L, d, V, 3, "classifier", lam=0.6, gamma=0.97, B=B)
        e = X.Engine(g, mega=True)
        e.set_option("lm_tail", k)
        e.session_begin(first, 60, 100, 5)
        e.decode_run(3)
        runs.append(e.records(0, 3))
        e.close()
    assert np.array_equal(runs[0]["output_layer"], runs[1]["output_layer"])
    assert np.array_equal(runs[0]["tokens"], runs[1]["tokens"])


def test_engine_run_across_pipelined_and_persistent_batches(port):
    """Engine::run at max_batch 128 with ragged output lengths: the decode batch shrinks from 128
    through the pipelined kernel's 64-row-halves range (65-128) into the persistent kernel's
    (<= 64) as sequences finish and are evicted. K/V of every layer (prompt and generated
    positions) and the tokens vs the oracle's fp64 run on the same requests."""
    L, d, V, B = 3, 256, 512, 128
    g = X.EngineConfig(model=X.ModelConfig(L, d, V, 29), technique=X.ExitTechnique("never"), max_batch=B,
                       pool_blocks=8192, eos_token=-1, capture_kv=True)
    o = OB.engine_config(L, d, V, 29, "never", max_batch=B, pool_blocks=8192, eos_token=-1, capture_kv=True,
                         round_bf16=True)
    rng = np.random.default_rng(4)
    reqs = [(0.0, [int(x) for x in rng.integers(1, V, 2 + i % 5)], 1 + (i * 5) % 9) for i in range(B)]
    e = X.Engine(g, mega=True)
    t = e.run(X.Workload([X.Request(*r) for r in reqs]))
    tp = port.model(L, d, V, 29, True).run(o, OB.Workload.from_requests(reqs))
    gt = {s["id"]: s["tokens"] for s in t.sequences}
    pt = {s["id"]: s["tokens"] for s in tp.sequences}
    assert all(len(gt[k]) == len(pt[k]) for k in pt)
    assert np.mean([a == b for k in pt for a, b in zip(gt[k], pt[k])]) >= 0.9
    for sid in range(0, B, 9):
        n = len(reqs[sid][1]) - 1
        for layer in range(1, L + 1):
            kg, vg = t.kv(sid, layer)
            ko, vo = port.transcript_kv(tp, sid, layer, d)
            assert relerr(kg[:n], ko[:n]) <= HID_TOL and relerr(vg[:n], vo[:n]) <= HID_TOL, (sid, layer)
    e.close()
