"""f3: transcript persistence in the reference's JSON-lines format (engine.cpp:336-461).
The writer is checked byte for byte against the reference's own write_transcript_jsonl
(oracle/_ref) on the same transcripts, and the reader round-trips it."""
import numpy as np
import pytest

from oracle import bindings as OB
from paper_2407_20272_b200 import exitlab as X

CASES = [("never", {}, {}), ("state", dict(lambda0=0.97, gamma=0.99), {}),
         ("always_at", dict(exit_layer=2), dict(exit_layer=2)), ("softmax", dict(lambda0=1e-3), {}),
         ("classifier", dict(lambda0=0.55), {})]


@pytest.mark.parametrize("tech,kw,tk", CASES)
def test_jsonl_byte_identical_to_reference(port, ref, tmp_path, tech, kw, tk):
    L, d, V = 3, 16, 32
    cfg = OB.engine_config(L, d, V, 11, tech, max_batch=3, pool_blocks=128, block_capacity=4, **kw)
    wl = port.gen_workload(n_requests=7, mean_interarrival=0.013, prompt_len_min=1, prompt_len_max=5,
                           output_len_min=1, output_len_max=6, seed=3, vocab_size=V)
    tr = ref.model(L, d, V, 11).run(cfg, wl)
    a, b = tmp_path / "ref.jsonl", tmp_path / "ours.jsonl"
    ref.write_transcript_jsonl(tr, str(a))
    X.write_transcript_jsonl(tr, str(b), X.ModelConfig(L, d, V, 11), X.ExitTechnique(tech, tk.get("exit_layer", 1)))
    assert a.read_bytes() == b.read_bytes()
    # the port's transcript of the same run is the same file (bit-exact port)
    tp = port.model(L, d, V, 11).run(cfg, wl)
    c = tmp_path / "port.jsonl"
    X.write_transcript_jsonl(tp, str(c), X.ModelConfig(L, d, V, 11), X.ExitTechnique(tech, tk.get("exit_layer", 1)))
    assert a.read_bytes() == c.read_bytes()


def test_jsonl_reader_round_trip_and_errors(port, tmp_path):
    L, d, V = 3, 16, 32
    cfg = OB.engine_config(L, d, V, 11, "state", lambda0=0.97, max_batch=3, pool_blocks=128, block_capacity=4)
    wl = OB.Workload.from_requests([(0.0, [1, 2], 3), (0.0, [3], 2)])
    tp = port.model(L, d, V, 11).run(cfg, wl)
    p = tmp_path / "t.jsonl"
    X.write_transcript_jsonl(tp, str(p), X.ModelConfig(L, d, V, 11), X.ExitTechnique("state"))
    r = X.read_transcript_jsonl(str(p))
    assert r["meta"]["n_layers"] == L and r["meta"]["technique"] == "state"
    assert [s["tokens"] for s in r["sequences"]] == [s["tokens"] for s in tp.sequences]
    assert np.allclose([it["clock"] for it in r["iterations"]], tp["it_clock"])
    bad = tmp_path / "bad.jsonl"
    bad.write_text('{"type":"bogus"}\n')
    with pytest.raises(RuntimeError):
        X.read_transcript_jsonl(str(bad))
    bad.write_text('{"type":"prefill","clock":0.0,"charge":0.0,"seq_id":0,"positions":1}\n')
    with pytest.raises(RuntimeError):
        X.read_transcript_jsonl(str(bad))
