"""T5 mode (north_star (1): cross-attention over encoder states) in the CPU
oracle.  The reference has no encoder or cross-attention, so
this mode's oracle is pinned here by an independent numpy restatement of the
decoder block with the extra sub-layer (self-attn residual -> cross-attn
residual -> ReLU MLP residual, norm-free like model.cpp:197-272), and by
encoder_len = 0 reducing exactly to the reference model."""
import numpy as np

from oracle import bindings as OB


def np_t5_decode(m, prompt, max_new, seq_id, T, heads=1):
    """token-by-token greedy decode (technique never) of the T5-mode model, fp64; heads > 1:
    self- and cross-attention per head of d / heads features, scale 1 / sqrt(d / heads)."""
    L, d = m.L, m.d
    W = {(n, l): m.tensor(n, l) for l in range(1, L + 1)
         for n in ("w_q", "w_k", "w_v", "w_o", "w_up", "w_down", "w_qc", "w_kc", "w_vc", "w_oc")}
    emb, lm = m.tensor("embedding"), m.tensor("lm_head")
    E = np.stack([m.encoder_state(seq_id, t) for t in range(T)])
    K = [[] for _ in range(L)]
    Vv = [[] for _ in range(L)]
    hd = d // heads
    sc = 1.0 / np.sqrt(hd)

    def softmax(x):
        e = np.exp(x - x.max())
        return e / e.sum()

    def attend(Km, Vm, q):  # Km, Vm [n][d]
        return np.concatenate([softmax(Km[:, f:f + hd] @ q[f:f + hd] * sc) @ Vm[:, f:f + hd]
                               for f in range(0, d, hd)])

    def layer(l, h):
        q, k, v = W["w_q", l] @ h, W["w_k", l] @ h, W["w_v", l] @ h
        K[l - 1].append(k)
        Vv[l - 1].append(v)
        mid = h + W["w_o", l] @ attend(np.array(K[l - 1]), np.array(Vv[l - 1]), q)
        qc = W["w_qc", l] @ mid
        kc, vc = E @ W["w_kc", l].T, E @ W["w_vc", l].T
        mid = mid + W["w_oc", l] @ attend(kc, vc, qc)
        return mid + W["w_down", l] @ np.maximum(W["w_up", l] @ mid, 0.0)

    for tok in prompt[:-1]:
        h = emb[tok].copy()
        for l in range(1, L + 1):
            h = layer(l, h)
    x, out = prompt[-1], []
    for _ in range(max_new):
        h = emb[x].copy()
        for l in range(1, L + 1):
            h = layer(l, h)
        x = int(np.argmax(lm @ h))
        out.append(x)
    return out


def test_t5_zero_encoder_is_the_reference_model(port):
    L, d, V = 3, 16, 32
    a, b = port.model(L, d, V, 11, True), port.model(L, d, V, 11, True, encoder_len=0)
    for n in ("embedding", "lm_head"):
        assert np.array_equal(a.tensor(n), b.tensor(n))
    cfg = OB.engine_config(L, d, V, 11, "never", max_batch=2, pool_blocks=64, block_capacity=4, round_bf16=True)
    wl = OB.Workload.from_requests([(0.0, [1, 2, 3], 5), (0.0, [4], 4)])
    ta, tb = a.run(cfg, wl), b.run(cfg, wl)
    assert np.array_equal(ta["ps_token"], tb["ps_token"])


def test_t5_engine_matches_numpy_restatement(port):
    L, d, V, T = 3, 16, 32, 5
    m = port.model(L, d, V, 11, True, encoder_len=T)
    cfg = OB.engine_config(L, d, V, 11, "never", max_batch=2, pool_blocks=64, block_capacity=4, round_bf16=True)
    reqs = [(0.0, [1, 2, 3], 6), (0.0, [7, 5], 4)]
    t = m.run(cfg, OB.Workload.from_requests(reqs))
    got = {s["id"]: s["tokens"] for s in t.sequences}
    for sid, (_, prompt, mx) in enumerate(reqs):
        assert got[sid] == np_t5_decode(m, prompt, mx, sid, T), sid
    # the cross sub-layer changes the model (different tokens than the decoder-only model somewhere)
    base = port.model(L, d, V, 11, True).run(cfg, OB.Workload.from_requests(reqs))
    assert any(x != y for s, r in zip(t.sequences, base.sequences) for x, y in zip(s["tokens"], r["tokens"])) or \
        not np.array_equal(t["it_conf"], base["it_conf"])


def test_encoder_states_are_seeded_and_bf16(port):
    m = port.model(2, 32, 64, 3, True, encoder_len=4)
    e = m.encoder_state(5, 2)
    assert np.array_equal(e, m.encoder_state(5, 2)) and not np.array_equal(e, m.encoder_state(5, 3))
    assert np.all(np.abs(e) <= 1.0 / np.sqrt(32))
    bits = e.astype(np.float32).view(np.uint32)
    assert np.all((bits & 0xFFFF) == 0)  # exactly representable in bf16


def test_t5_multi_head_matches_numpy_restatement(port):
    L, d, V, T = 3, 32, 48, 5
    reqs = [(0.0, [1, 2, 3], 6), (0.0, [7, 5], 4)]
    cfg = OB.engine_config(L, d, V, 11, "never", max_batch=2, pool_blocks=64, block_capacity=4, round_bf16=True)
    toks = {}
    for heads in (1, 4):
        m = port.model(L, d, V, 11, True, encoder_len=T, n_heads=heads)
        t = m.run(cfg, OB.Workload.from_requests(reqs))
        got = {s["id"]: s["tokens"] for s in t.sequences}
        for sid, (_, prompt, mx) in enumerate(reqs):
            assert got[sid] == np_t5_decode(m, prompt, mx, sid, T, heads), (heads, sid)
        toks[heads] = t["it_conf"]
    assert not np.array_equal(toks[1], toks[4])  # the head split changes the model


def test_multi_head_needs_a_divisor(port):
    import pytest
    with pytest.raises(ValueError):
        port.model(2, 32, 48, 1, True, encoder_len=4, n_heads=5)


def np_encoder(m, seq_id, T, heads=1):
    """independent numpy restatement of the T5 encoder stack: bidirectional norm-free blocks over
    the embeddings of the seeded encoder ids, output bf16-rounded like the model"""
    d = m.d
    hd = d // heads
    emb = m.tensor("embedding")
    X = np.stack([emb[m.encoder_token(seq_id, t)] for t in range(T)])
    for l in range(1, m.encoder_layers + 1):
        W = {n: m.tensor(n, l) for n in ("e_q", "e_k", "e_v", "e_o", "e_up", "e_down")}
        Q, K, Vv = X @ W["e_q"].T, X @ W["e_k"].T, X @ W["e_v"].T
        A = np.zeros_like(X)
        for f in range(0, d, hd):
            S = Q[:, f:f + hd] @ K[:, f:f + hd].T / np.sqrt(hd)
            P = np.exp(S - S.max(axis=1, keepdims=True))
            A[:, f:f + hd] = (P / P.sum(axis=1, keepdims=True)) @ Vv[:, f:f + hd]
        mid = X + A @ W["e_o"].T
        X = mid + np.maximum(mid @ W["e_up"].T, 0.0) @ W["e_down"].T
    b = np.ascontiguousarray(X, dtype=np.float64).view(np.uint64)  # RNE to 8 significant bits on fp64 bits
    b = (b + np.uint64((1 << 44) - 1) + ((b >> np.uint64(45)) & np.uint64(1))) & ~np.uint64((1 << 45) - 1)
    return b.view(np.float64)


def test_t5_encoder_stack_matches_numpy(port):
    L, d, V, T = 2, 32, 48, 6
    for heads, nl in ((1, 2), (4, 3)):
        m = port.model(L, d, V, 11, True, encoder_len=T, n_heads=heads, encoder_layers=nl)
        for sid in (0, 3):
            want = np_encoder(m, sid, T, heads)
            got = np.stack([m.encoder_state(sid, t) for t in range(T)])
            assert np.abs(got - want).max() <= 2 ** -8 * np.abs(want).max(), (heads, sid)  # one bf16 ulp
        ids = [m.encoder_token(0, t) for t in range(T)]
        assert all(1 <= i < V for i in ids) and len(set(ids)) > 1
    # the stack changes the states, and the decode (vs seeded states)
    m0 = port.model(L, d, V, 11, True, encoder_len=T)
    m2 = port.model(L, d, V, 11, True, encoder_len=T, encoder_layers=2)
    assert not np.allclose(m0.encoder_state(1, 2), m2.encoder_state(1, 2))
    cfg = OB.engine_config(L, d, V, 11, "never", max_batch=2, pool_blocks=64, block_capacity=4, round_bf16=True)
    reqs = [(0.0, [1], 6), (0.0, [7], 4)]
    t2 = m2.run(cfg, OB.Workload.from_requests(reqs))
    got = {s["id"]: s["tokens"] for s in t2.sequences}
    assert got[0] == np_t5_decode(m2, [1], 6, 0, T) and got[1] == np_t5_decode(m2, [7], 4, 1, T)
