"""The N>1 path on CPU: world_size-2 gloo processes shard requests and all-gather
per-(request, SSM) acceptance statistics exactly as bench.py does over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_15921_b200.dist import AcceptanceStats, shard


def test_shard_partitions_requests():
    for n in (1, 7, 32, 256):
        for w in (1, 2, 3, 4, 8):
            ids = [i for r in range(w) for i in shard(n, w, r)]
            assert ids == list(range(n))
            sizes = [len(shard(n, w, r)) for r in range(w)]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_req, n_ssm, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    st = AcceptanceStats(n_req, n_ssm, world, rank)
    for step in range(3):
        for li, rid in enumerate(st.owned):
            st.add(li, rid % n_ssm, float(rid * 10 + step))
    g = st.gather(dist)
    q.put((rank, g.numpy().tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_req", [7, 32])
def test_gloo_allgather_of_acceptance_stats(n_req):
    world, n_ssm = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_req, n_ssm, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # identical on every rank, and equal to the single-process reference
    assert res[0] == res[1]
    ref = torch.zeros((n_req, n_ssm, 2), dtype=torch.float64)
    for rid in range(n_req):
        for step in range(3):
            ref[rid, rid % n_ssm, 0] += rid * 10 + step
            ref[rid, rid % n_ssm, 1] += 1
    assert torch.equal(torch.tensor(res[0], dtype=torch.float64), ref)
    means = AcceptanceStats.means(ref)
    assert torch.isinf(means[0, 1]) and means[1, 1] == 10 + 1


def test_add_many_matches_add():
    a = AcceptanceStats(10, 3, 1, 0)
    b = AcceptanceStats(10, 3, 1, 0)
    rng = np.random.default_rng(7)
    idx, ssm, gp = rng.integers(0, 10, 50), rng.integers(0, 3, 50), rng.random(50)
    for i, j, g in zip(idx, ssm, gp):
        a.add(int(i), int(j), float(g))
    b.add_many(idx, ssm, gp)
    assert torch.allclose(a.gather(), b.gather())
