"""Quick on-box smoke of the CUDA path against the oracle port (debug helper)."""
import sys, time, traceback
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2407_20272_b200 import exitlab as X
from oracle import bindings as OB

P = OB.port()

def step(name, fn):
    t = time.time()
    try:
        r = fn()
        print(f"[ok] {name} ({time.time()-t:.2f}s) {r if r is not None else ''}", flush=True)
    except Exception as e:
        print(f"[FAIL] {name}: {e}", flush=True)
        traceback.print_exc()

def mk(L, d, V, seed, tech="never", **kw):
    cfg = X.EngineConfig(model=X.ModelConfig(L, d, V, seed), technique=X.ExitTechnique(tech, kw.pop("exit_layer", 1)),
                         schedule=X.ThresholdSchedule(kw.pop("lambda0", 0.85), kw.pop("gamma", 1.0), 0.0), **kw)
    return cfg

graph = int(sys.argv[1]) if len(sys.argv) > 1 else 0

def t_weights():
    cfg = mk(3, 8, 16, 11, max_batch=4, pool_blocks=256, block_capacity=4)
    e = X.Engine(cfg, graph=bool(graph))
    m = P.model(3, 8, 16, 11, round_bf16=True)
    bad = []
    for name in ["embedding", "lm_head", "w_q", "w_k", "w_v", "w_o", "w_up", "w_down", "probe_w", "probe_b"]:
        for layer in ([1, 3] if name.startswith("w_") else [0]):
            g = X.bf16_to_f64(e.model_tensor(name, layer)).ravel()
            o = m.tensor(name, layer).ravel()
            if not np.array_equal(g, o):
                bad.append((name, layer, np.abs(g-o).max()))
    assert not bad, bad
    e.close()

def t_run_never():
    cfg = mk(3, 8, 16, 11, max_batch=4, pool_blocks=256, block_capacity=4, eos_token=-1)
    e = X.Engine(cfg, graph=bool(graph))
    wl = X.Workload([X.Request(0.0, [1, 2, 3], 6)])
    t = e.run(wl)
    m = P.model(3, 8, 16, 11, round_bf16=True)
    ref = m.reference_decode([1, 2, 3], 6, -1)
    return dict(gpu=t.sequences[0]["tokens"], oracle=ref, layers=t["it_output_layer"].tolist())

def t_session(L=12, d=768, B=8, tech="state", lam=0.95):
    cfg = mk(L, d, 32128, 0, tech, lambda0=lam, max_batch=B, pool_blocks=B*L*40, block_capacity=16, eos_token=-1)
    e = X.Engine(cfg, graph=bool(graph))
    first = (np.arange(B) * 7 + 3).astype(np.int32)
    e.session_begin(first, 64, 80, 99)
    ocfg = OB.engine_config(L, d, 32128, 0, tech, lambda0=lam, max_batch=B, pool_blocks=B*L*40, block_capacity=16, eos_token=-1, round_bf16=True)
    m = P.model(L, d, 32128, 0, round_bf16=True)
    s = m.session(ocfg, first, 64, 80, 99)
    out = []
    for it in range(3):
        g = e.decode_iteration()
        o = s.step(forced=g["output_layer"])
        hg = e.hidden(g["output_layer"] & 1)
        err = np.abs(hg - o["h_exit"]).max() / np.abs(o["h_exit"]).max()
        out.append(dict(e=g["output_layer"], e_oracle_forced=o["output_layer"], tok_agree=float((g["tokens"] == o["tokens"]).mean()),
                        h_relerr=float(err), conf_g=g["conf"][0][:3].tolist(), conf_o=o["conf"][0][:3].tolist()))
    t0 = time.time(); ms = e.time_decode(5); 
    out.append(dict(ms_per_iter=ms/5))
    e.close()
    return out

step("weights bit-exact", t_weights)
step("run never tiny", t_run_never)
step("session C1-ish state", lambda: t_session(6, 512, 8, "state", 0.95))
step("session C2 state", lambda: t_session(12, 768, 64, "state", 0.97))
step("session softmax", lambda: t_session(6, 512, 8, "softmax", 1e-7))
