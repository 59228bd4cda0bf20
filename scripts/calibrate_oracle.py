"""Threshold calibration on the oracle (CPU): full-depth confidences of the bench workload.

    python scripts/calibrate_oracle.py L d B tech iters target_e

Runs the oracle's decode session (gen_workload(seed 1) prompts, seeded 511-position KV
prefix) with a threshold no sequence reaches, so every layer's confidence is computed, then
searches lambda0 (for a few gammas) so that the batch-barrier exit layer
max_b first_accept_b averages target_e.  An estimate: the real run's later iterations
attend over filled K/V of skipped layers, so the chosen schedule is re-measured by
tests/test_gpu_free_running.py and bench.py (which report the realised mean exit layer).
"""
import json
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from oracle import bindings as OB  # noqa: E402

V = 32128


def confidences(L, d, B, tech, iters):
    port = OB.port()
    m = port.model(L, d, V, 0, True)
    never_lam = {"state": 2.0, "classifier": 2.0, "softmax": 2.0}[tech]
    cfg = OB.engine_config(L, d, V, 0, tech, lambda0=never_lam, gamma=1.0, max_batch=B, pool_blocks=4096,
                           eos_token=-1, round_bf16=True)
    wl = port.gen_workload(n_requests=B, prompt_len_min=512, prompt_len_max=512, output_len_min=128,
                           output_len_max=128, seed=1, vocab_size=V)
    first = wl.prompt[wl.prompt_off[1:] - 1]
    s = m.session(cfg, first, 511, 640, 1, np.arange(B))
    return np.stack([s.step()["conf"] for _ in range(iters)])  # [it][L][B]


def exit_layers(conf, lam0, gamma):
    L = conf.shape[1]
    lam = np.array([max(0.0, lam0 * gamma ** l) for l in range(L)])
    acc = conf > lam[None, :, None]
    first = np.where(acc.any(axis=1), acc.argmax(axis=1) + 1, L)  # [it][B]
    return first.max(axis=1)


if __name__ == "__main__":
    L, d, B, tech, iters, target = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4],
                                    int(sys.argv[5]), float(sys.argv[6]))
    c = confidences(L, d, B, tech, iters)
    out = {"L": L, "d": d, "B": B, "tech": tech,
           "p10_p50_p90_by_layer": [[float(np.quantile(c[:, l], q)) for q in (0.1, 0.5, 0.9)] for l in range(L)],
           "best": []}
    for gamma in (1.0, 0.999, 0.997, 0.995, 0.99, 0.98):
        lo, hi = float(np.min(c)) * 0.5, float(np.max(c)) * 2.0
        for _ in range(80):  # mean exit layer is non-increasing... in lambda0 -> bisection
            mid = 0.5 * (lo + hi)
            if exit_layers(c, mid, gamma).mean() > target:
                hi = mid
            else:
                lo = mid
        e = exit_layers(c, hi, gamma)
        out["best"].append({"gamma": gamma, "lambda0": hi, "mean_e": float(e.mean()), "e": e.tolist()})
    print(json.dumps(out))
