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
