"""The sub-engine C ABI (el_kv_*, el_layer_forward, el_kv_fill, el_exit_confidence,
el_greedy_tokens) against the reference's semantics.

* KvStore (kv_cache.hpp:45-75): test_kv_cache.cpp's cases on the device pool -- reservation
  arithmetic, OOM without leak, write-once / contiguity, capacity, view bounds, commit
  completeness, release, and conservation of blocks under random operations; the error
  classes are the reference's (ValueError = invalid_argument, RuntimeError = runtime_error,
  KvOutOfMemory).
* layer_forward (model.cpp:197-272), fill_skipped + compute_kv_pair (kv_cache.cpp:222-234,
  model.cpp:274-282), the three confidences + decide (exit_policy.cpp:57-115) and greedy_token
  (model.cpp:288-299) against fp64 restatements on the same bf16 weights (numpy, the
  reference's loop semantics), within the bf16 tolerances of the engine-level parity tests.
"""
import numpy as np
import pytest

from oracle import bindings as OB
from paper_2407_20272_b200 import exitlab as X

pytestmark = pytest.mark.gpu

TOL = 8e-3


def relerr(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-30))


def bf16(x):
    a = np.asarray(x, np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16 << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def engine(L=4, d=128, V=512, tech="never", lam=0.5, gamma=1.0, B=8, pool=512, bc=16, seed=3):
    cfg = X.EngineConfig(model=X.ModelConfig(L, d, V, seed), technique=X.ExitTechnique(tech, 2),
                         schedule=X.ThresholdSchedule(lam, gamma, 0.0), max_batch=B, pool_blocks=pool,
                         block_capacity=bc, eos_token=-1)
    return X.Engine(cfg)


def test_kvstore_semantics_on_device():
    e = engine(L=3, d=64, pool=40, bc=4)
    kv = e.kv_store()
    kv.allocate(7, 10)  # ceil(10/4) = 3 blocks per layer x 3 layers (test_kv_cache.cpp:18-27)
    assert kv.stats()["free_blocks"] == 40 - 9
    with pytest.raises(ValueError):
        kv.allocate(7, 4)  # duplicate id
    with pytest.raises(ValueError):
        kv.allocate(8, -1)
    with pytest.raises(X.KvOutOfMemory):
        kv.allocate(9, 4 * 11)  # 33 blocks > 31 free
    assert kv.stats()["free_blocks"] == 31  # no leak on OOM (test_kv_cache.cpp:29-33)
    rng = np.random.default_rng(0)
    k0, v0 = rng.standard_normal(64), rng.standard_normal(64)
    kv.append(7, 1, 0, k0, v0)
    with pytest.raises(RuntimeError):
        kv.append(7, 1, 0, k0, v0)  # overwrite
    with pytest.raises(RuntimeError):
        kv.append(7, 1, 2, k0, v0)  # gap
    with pytest.raises(ValueError):
        kv.append(7, 4, 0, k0, v0)  # layer outside [1, L]
    with pytest.raises(ValueError):
        kv.append(99, 1, 0, k0, v0)  # unknown seq
    k, v = kv.view(7, 1, 1)
    assert np.array_equal(k[0], bf16(k0)) and np.array_equal(v[0], bf16(v0))  # bf16 storage, exact
    with pytest.raises(RuntimeError):
        kv.view(7, 2, 1)  # nothing written at layer 2
    with pytest.raises(RuntimeError):
        kv.commit(7)  # layers 2, 3 incomplete (test_kv_cache.cpp:80-89)
    for layer in (2, 3):
        kv.append(7, layer, 0, k0, v0)
    kv.commit(7)
    assert kv.committed_len(7) == 1 and kv.written_len(7, 2) == 1
    for p in range(1, 12):
        for layer in (1, 2, 3):
            kv.append(7, layer, p, k0 * p, v0)
        kv.commit(7)
    with pytest.raises(X.KvOutOfMemory):
        kv.append(7, 1, 12, k0, v0)  # reserved capacity = 12 positions
    kv.release(7)
    with pytest.raises(ValueError):
        kv.release(7)
    assert kv.stats()["free_blocks"] == 40
    # conservation under random allocate / release (test_kv_cache.cpp:108-145)
    live = {}
    for i in range(60):
        if live and (rng.random() < 0.45 or len(live) == 8):
            sid = int(rng.choice(list(live)))
            kv.release(sid)
            del live[sid]
        else:
            sid, cap = 100 + i, int(rng.integers(0, 14))
            try:
                kv.allocate(sid, cap)
                live[sid] = -(-cap // 4) * 3
            except X.KvOutOfMemory:
                pass
        assert kv.stats()["free_blocks"] == 40 - sum(live.values())
    e.close()


def _ref_layer(m, layer, h, K, V):
    """model.cpp:197-272 in fp64 for one sequence: h (fp32) -> out; K/V: cached rows incl. the new one."""
    d = h.shape[0]
    hb = bf16(h)  # the device feeds the tensor cores bf16 operands
    q = m.tensor("w_q", layer) @ hb
    s = K @ q / np.sqrt(d)
    p = np.exp(s - s.max())
    p /= p.sum()
    att = p @ V
    mid = h + m.tensor("w_o", layer) @ bf16(att)
    up = np.maximum(m.tensor("w_up", layer) @ bf16(mid), 0.0)
    return mid + m.tensor("w_down", layer) @ bf16(up)


def test_layer_forward_fill_and_heads_vs_fp64(port):
    L, d, V = 4, 128, 512
    e = engine(L, d, V)
    m = port.model(L, d, V, 3, True)
    kv = e.kv_store()
    rng = np.random.default_rng(1)
    ids, P = [5, 9, 2], [3, 0, 17]
    for sid, n in zip(ids, P):
        kv.allocate(sid, 40)
        for p in range(n):
            for layer in range(1, L + 1):
                kv.append(sid, layer, p, rng.standard_normal(d) * 0.3, rng.standard_normal(d) * 0.3)
            kv.commit(sid)
    h = [rng.standard_normal(d).astype(np.float32) * 0.5 for _ in ids]
    # layers 1..2 computed, 3..4 filled from the layer-2 state (an exit at 2)
    for layer in (1, 2):
        out = X.layer_forward(e, layer, list(zip(ids, h)))
        for i, sid in enumerate(ids):
            K, Vv = kv.view(sid, layer, P[i] + 1)
            kq = m.tensor("w_k", layer) @ bf16(h[i])
            vq = m.tensor("w_v", layer) @ bf16(h[i])
            assert relerr(K[-1], kq) <= TOL and relerr(Vv[-1], vq) <= TOL  # appended K/V
            want = _ref_layer(m, layer, h[i].astype(np.float64), K.astype(np.float64), Vv.astype(np.float64))
            assert relerr(out[i], want) <= TOL, (layer, sid)
        h = out
    with pytest.raises(RuntimeError):
        X.layer_forward(e, 2, [(ids[0], h[0])])  # layer 2 already holds this position
    with pytest.raises(ValueError):
        X.fill_skipped(e, [(ids[0], h[0])], L + 1)
    X.fill_skipped(e, list(zip(ids, h)), 2)
    for i, sid in enumerate(ids):
        for layer in (3, 4):
            K, Vv = kv.view(sid, layer, P[i] + 1)
            assert relerr(K[-1], m.tensor("w_k", layer) @ bf16(h[i])) <= TOL
            assert relerr(Vv[-1], m.tensor("w_v", layer) @ bf16(h[i])) <= TOL
        kv.commit(sid)  # every layer now holds the position (kv_cache.cpp:165-180)
    X.fill_skipped(e, list(zip(ids, h)), L)  # no-op at the last layer
    # greedy_token over the LM head (lowest index on ties)
    toks = X.greedy_tokens(e, np.stack(h))
    lm = m.tensor("lm_head")
    for i in range(len(ids)):
        lg = lm @ bf16(h[i])
        top2 = np.sort(lg)[-2:]
        assert toks[i] == int(np.argmax(lg)) or top2[1] - top2[0] < 2e-2
    e.close()


@pytest.mark.parametrize("tech,lam", [("state", 0.9), ("classifier", 0.5), ("softmax", 0.003), ("always_at", 0.5),
                                      ("never", 0.5)])
def test_exit_confidence_and_decide(port, tech, lam):
    L, d, V = 4, 128, 512
    e = engine(L, d, V, tech, lam=lam, gamma=0.99)
    m = port.model(L, d, V, 3, True)
    rng = np.random.default_rng(2)
    hp = rng.standard_normal((6, d)).astype(np.float32)
    hc = (hp + 0.4 * rng.standard_normal((6, d))).astype(np.float32)
    for layer in (1, 3):
        lam_l = port.threshold_at(lam, 0.99, 0.0, layer)
        conf, acc = X.exit_confidence(e, layer, hc, hp)
        for b in range(6):
            if tech == "state":
                want = port.state_similarity(hp[b].astype(np.float64), hc[b].astype(np.float64))
                assert abs(conf[b] - want) <= 1e-6
            elif tech == "classifier":
                want = port.classifier(hc[b].astype(np.float64), m.tensor("probe_w"), float(m.tensor("probe_b")[0]))
                assert abs(conf[b] - want) <= 1e-6
            elif tech == "softmax":
                want = port.softmax_response(m.tensor("lm_head") @ bf16(hc[b]))
                assert abs(conf[b] - want) <= 1e-4 * max(want, 1e-3)
            if tech in ("state", "classifier", "softmax"):
                assert acc[b] == (float(conf[b]) > lam_l)  # strict '>' (exit_policy.cpp:89-115)
            elif tech == "always_at":
                assert acc[b] == (layer >= 2)
            else:
                assert not acc[b]
    e.close()


def test_subengine_rejected_during_a_session():
    e = engine()
    e.session_begin(np.arange(4) + 1, 8, 20, 1)
    with pytest.raises(X.LogicError):
        e.kv_store().allocate(1, 4)
    e.session_end()
    e.kv_store().allocate(1, 4)  # fine once the session is over
    e.close()


@pytest.mark.parametrize("heads", [4, 16])
def test_layer_forward_multi_head_sharp_attention(port, heads):
    """The head split (extension: CALM-T5 attention; the reference has one head) with SHARP
    attention: large cached keys make each head's softmax peak on different positions, so a
    single softmax over d features would give a different output.  Per-head fp64 reference."""
    L, d, V = 2, 128, 256
    hd = d // heads
    e = X.Engine(X.EngineConfig(model=X.ModelConfig(L, d, V, 3, n_heads=heads), technique=X.ExitTechnique("never"),
                                max_batch=8, pool_blocks=256, eos_token=-1))
    m = port.model(L, d, V, 3, True)
    kv = e.kv_store()
    rng = np.random.default_rng(7)
    ids, P = [1, 4], [9, 21]
    for sid, n in zip(ids, P):
        kv.allocate(sid, 40)
        for p in range(n):
            for layer in range(1, L + 1):
                kv.append(sid, layer, p, rng.standard_normal(d) * 4.0, rng.standard_normal(d))
            kv.commit(sid)
    h = [rng.standard_normal(d).astype(np.float32) * 2.0 for _ in ids]
    out = X.layer_forward(e, 1, list(zip(ids, h)))
    for i, sid in enumerate(ids):
        K, Vv = kv.view(sid, 1, P[i] + 1)
        K, Vv = K.astype(np.float64), Vv.astype(np.float64)
        hb = bf16(h[i].astype(np.float64))
        q = m.tensor("w_q", 1) @ hb
        att = np.zeros(d)
        for f in range(0, d, hd):
            s = K[:, f:f + hd] @ q[f:f + hd] / np.sqrt(hd)
            p = np.exp(s - s.max())
            att[f:f + hd] = (p / p.sum()) @ Vv[:, f:f + hd]
        s1 = K @ q / np.sqrt(d)
        p1 = np.exp(s1 - s1.max())
        att1 = (p1 / p1.sum()) @ Vv
        assert relerr(att1, att) > 0.2  # the heads genuinely attend differently
        mid = h[i] + m.tensor("w_o", 1) @ bf16(att)
        want = mid + m.tensor("w_down", 1) @ bf16(np.maximum(m.tensor("w_up", 1) @ bf16(mid), 0.0))
        assert relerr(out[i], want) <= TOL, (heads, sid, relerr(out[i], want))
        mid1 = h[i] + m.tensor("w_o", 1) @ bf16(att1)
        want1 = mid1 + m.tensor("w_down", 1) @ bf16(np.maximum(m.tensor("w_up", 1) @ bf16(mid1), 0.0))
        assert relerr(out[i], want) < relerr(out[i], want1) / 3
    e.close()
