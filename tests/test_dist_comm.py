"""The N>1 exchange through the C ABI on CPU: world_size-2 processes shard requests
and all-gather per-(request, SSM) ArmEstimate rows with spin_stats_allgather (TCP
transport: the NCCL transport's semantics without a GPU), then feed the gathered
rows into the C++ LBSS on every rank -- both ranks must derive identical estimates
and identical assignments."""
import multiprocessing as mp

import numpy as np
import pytest

from paper_2503_15921_b200 import dist
from paper_2503_15921_b200.dist import TCP, AcceptanceStats, Comm, shard


def test_shard_partitions_requests():
    for n in (1, 7, 32, 256):
        for w in (1, 2, 3, 4, 8):
            ids = [i for r in range(w) for i in shard(n, w, r)]
            assert ids == list(range(n))
            sizes = [len(shard(n, w, r)) for r in range(w)]
            assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, uid, n_req, n_ssm, q):
    from paper_2503_15921_b200.selector import Lbss

    comm = Comm(TCP, rank, world, uid)
    st = AcceptanceStats(n_req, n_ssm, world, rank)
    sel = Lbss(n_req, [n_req] * n_ssm, alpha=4, beta=2, seed=5)
    plans = []
    for step in range(6):
        a, _ = sel.next_slot()
        plans.append(a.tolist())
        for li, rid in enumerate(st.owned):
            if a[rid] >= 0:
                st.add(li, int(a[rid]), float(rid * 10 + step + a[rid]))
        g = st.gather(comm)
        sel.set_rows(g)
    mx = comm.max(float(rank + 1))
    sm = comm.sum(float(rank + 1))
    comm.barrier()
    q.put((rank, g.tolist(), plans, mx, sm))
    comm.close()


@pytest.mark.parametrize("n_req,world", [(7, 2), (32, 2), (9, 3)])
def test_c_abi_allgather_feeds_identical_selectors(n_req, world):
    n_ssm = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    uid = dist.unique_id(TCP)
    procs = [ctx.Process(target=_worker, args=(r, world, uid, n_req, n_ssm, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        rank, g, plans, mx, sm = q.get(timeout=120)
        res[rank] = (g, plans, mx, sm)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(1, world):
        assert res[r][0] == res[0][0] and res[r][1] == res[0][1]  # identical rows and plans on every rank
    assert all(res[r][2] == world and res[r][3] == world * (world + 1) / 2 for r in range(world))
    # the single-process reference: every request observed by the global plans
    ref = np.zeros((n_req, n_ssm, 2))
    for step, a in enumerate(res[0][1]):
        for rid in range(n_req):
            if a[rid] >= 0:
                ref[rid, a[rid], 0] += rid * 10 + step + a[rid]
                ref[rid, a[rid], 1] += 1
    assert np.array_equal(np.array(res[0][0]), ref)


def test_add_many_matches_add():
    a = AcceptanceStats(10, 3, 1, 0)
    b = AcceptanceStats(10, 3, 1, 0)
    rng = np.random.default_rng(7)
    idx, ssm, gp = rng.integers(0, 10, 50), rng.integers(0, 3, 50), rng.random(50)
    for i, j, g in zip(idx, ssm, gp):
        a.add(int(i), int(j), float(g))
    b.add_many(idx, ssm, gp)
    assert np.allclose(a.gather(), b.gather())
    means = AcceptanceStats.means(a.gather())
    assert np.isinf(means).any() or (a.gather()[..., 1] > 0).all()
