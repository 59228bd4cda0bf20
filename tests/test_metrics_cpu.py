"""f3: compute_metrics + write_report/read_report (metrics.cpp:13-210).

compute_metrics runs natively in libexitlab_b200 (el_metrics_compute, no device call) over a
transcript of the oracle port (bit-identical to the reference's own Engine::run); the reports
written by paper_2407_20272_b200.exitlab.write_report must be byte-identical to the
reference's write_report of the reference's transcript (wall_clock_info_s pinned to 0)."""
import numpy as np
import pytest

from oracle import bindings as B
from paper_2407_20272_b200 import exitlab as X

CASES = [("always_at", dict(exit_layer=4), 3), ("state", dict(lambda0=0.90), 4), ("softmax", dict(lambda0=0.02), 5),
         ("classifier", dict(lambda0=0.55, gamma=0.97), 6), ("never", {}, 7)]


@pytest.mark.parametrize("tech,kw,i", CASES)
def test_metrics_and_reports_match_reference(port, ref, tmp_path, tech, kw, i):
    cfg = B.engine_config(8, 64, 256, 1000 + i, tech, max_batch=8, pool_blocks=4096, eos_token=3, round_bf16=False,
                          **kw)
    wl = port.gen_workload(n_requests=10, mean_interarrival=0.01, prompt_len_min=1, prompt_len_max=9,
                           output_len_min=1, output_len_max=24, seed=40 + i, vocab_size=256, eos_token=3)
    tp = port.model(8, 64, 256, 1000 + i).run(cfg, wl)
    tr = ref.model(8, 64, 256, 1000 + i).run(cfg, wl)
    m = X.compute_metrics(tp, n_layers=8)
    assert m.total_tokens == len(tp["sq_tokens"]) and m.iterations == len(tp["it_output_layer"])
    assert sum(m.exit_layer_histogram) == m.total_tokens == sum(m.accept_layer_histogram)
    for fmt in ("json", "csv"):
        ours, theirs = tmp_path / f"ours.{fmt}", tmp_path / f"ref.{fmt}"
        X.write_report(m, str(ours), fmt)
        ref.write_report(tr, str(theirs), fmt, 0.0)
        assert ours.read_bytes() == theirs.read_bytes(), (fmt, ours.read_text(), theirs.read_text())
        back = X.read_report(str(theirs), fmt)
        assert back == m


def test_metrics_errors(port, tmp_path):
    cfg = B.engine_config(4, 16, 32, 1, "never", max_batch=4, pool_blocks=512, eos_token=-1)
    wl = port.gen_workload(n_requests=3, prompt_len_min=1, prompt_len_max=3, output_len_min=2, output_len_max=4,
                           seed=2, vocab_size=32)
    t = port.model(4, 16, 32, 1).run(cfg, wl)
    f = {k: np.array(t[k]) for k in ("it_output_layer", "it_batch_off", "sq_id", "sq_tok_off", "sq_exit_layers",
                                      "sq_first", "sq_finish", "meta")}
    f["sq_finish"][1] = -1.0  # an unfinished sequence (metrics.cpp:26-29)
    with pytest.raises(ValueError, match="unfinished"):
        X.compute_metrics(f, n_layers=4)
    with pytest.raises(ValueError):
        X.write_report(X.MetricsReport(), str(tmp_path / "r.txt"), "xml")
    (tmp_path / "bad.csv").write_text("metric,value\nthroughput_tokens_per_s,1\n")
    with pytest.raises(ValueError, match="missing metric"):
        X.read_report(str(tmp_path / "bad.csv"), "csv")
