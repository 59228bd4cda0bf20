"""bench.py host logic on the CPU: the synthetic workload equals the reference's
gen_workload, and the N>1 path (request sharding + max-over-ranks timing) works
as a 2-process gloo group."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def test_workload_matches_reference_gen_workload(port):
    w = port.gen_workload(n_requests=6, prompt_len_min=512, prompt_len_max=512, output_len_min=128,
                          output_len_max=128, seed=1, vocab_size=32128)
    p = bench.workload(6)
    for i in range(6):
        assert w.prompt[w.prompt_off[i]:w.prompt_off[i + 1]].tolist() == p[i]


def test_iteration_bytes_model():
    # full depth at C2, ctx 576 -> ~1580 MB
    b = bench.iteration_bytes(12, 768, 12, 576 * 64, 64, "never")
    assert abs(b / 1e6 - 1580.6) < 5.0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids = bench.shard(rank, world, 4)
    t = bench.reduce_max(float(10 + rank), dist)  # each rank's "time"; rank 1 is slower
    q.put((rank, ids, t))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_gloo_sharding_and_max_time():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=90) for _ in range(world))
    for p in ps:
        p.join(timeout=30)
    ids = [r[1] for r in res]
    assert ids[0] == [0, 1, 2, 3] and ids[1] == [4, 5, 6, 7]  # disjoint, covering, contiguous
    assert all(r[2] == 11.0 for r in res)  # max over ranks on every rank


@pytest.mark.timeout(300)
def test_bench_self_launches_two_ranks_and_reports():
    """`python bench.py --gpus 2` re-launches itself under torchrun (one rank per device), shards
    the requests, takes the max over ranks and prints ONE JSON line from rank 0 -- exercised with
    the CPU stub engine (EL_BENCH_STUB=1) over gloo."""
    import json
    import subprocess
    import sys
    env = dict(os.environ, EL_BENCH_STUB="1")
    r = subprocess.run([sys.executable, os.path.join(bench.ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
                        "--warmup", "3", "--config", "c2"], capture_output=True, text=True, env=env, timeout=280)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["config"]["global_batch"] == 128 and j["scaling"] == "weak"
    # stub: rank r takes 3 * (1 + 0.1 r) ms for 3 steps -> max over ranks = 3.3 ms
    assert abs(j["value"] - 64 * 2 * 3 / 3.3e-3) < 1.0
    assert j["layers_per_token"] == 6 and j["metrics"]["early_exit_rate_pct"] == 100.0
    assert j["full_layer"]["layers_per_token"] == 12


def test_bench_rejects_world_size_mismatch():
    import subprocess
    import sys
    env = dict(os.environ, EL_BENCH_STUB="1", WORLD_SIZE="1", RANK="0")
    r = subprocess.run([sys.executable, os.path.join(bench.ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
                        "--warmup", "3"], capture_output=True, text=True, env=env, timeout=60)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr
