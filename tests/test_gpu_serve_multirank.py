"""The native multi-rank serving loop (spin_lbss_serve, csrc/serve.cpp) on the GPU:
two ranks on one device (the NCCL transport needs one GPU per rank; the TCP
transport has the same gather semantics), each serving its contiguous shard of
the requests with the replicated C++ LBSS selector and a per-slot
spin_stats_allgather. Every rank must end with the same estimates and the same
plan, and its shard's requests must all have been served."""
import ctypes as C
import multiprocessing as mp

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N, SLOTS = 12, 14


def _rank(rank, world, uid, q):
    from paper_2503_15921_b200 import _lib
    from paper_2503_15921_b200.dist import TCP, Comm, shard
    from paper_2503_15921_b200.models import TINY_SSMS, TINY_TARGET, Engine, synthetic_prompts
    from paper_2503_15921_b200.selector import Lbss

    mine = shard(N, world, rank)
    prompts = synthetic_prompts(N, 16, 48, TINY_TARGET.vocab, 99)
    eng = Engine(TINY_TARGET, TINY_SSMS, max_requests=len(mine), max_ctx=256, window=4)
    eng.prefill(range(len(mine)), [prompts[i] for i in mine])
    comm = Comm(TCP, rank, world, uid)
    sel = Lbss(N, [N, N], alpha=4, beta=2, seed=7)
    rep = _lib.ServeReport()
    plan = np.zeros(N, np.int32)
    slots = np.arange(len(mine), dtype=np.int32)
    _lib.check(eng.lib.spin_lbss_serve(eng.ctx, comm.h, sel.h, N, 2, slots.ctypes.data_as(_lib.P_I32), len(mine),
                                       SLOTS, 1, C.byref(rep), plan.ctypes.data_as(_lib.P_I32)))
    committed = [len(eng.tokens(s)) for s in range(len(mine))]
    q.put((rank, sel.rows().tolist(), plan.tolist(), rep.tokens, rep.served, committed,
           [len(p) for p in (prompts[i] for i in mine)]))
    sel.close()
    comm.close()
    eng.close()


def test_two_ranks_serve_with_identical_selectors():
    from paper_2503_15921_b200 import dist

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    uid = dist.unique_id(dist.TCP)
    procs = [ctx.Process(target=_rank, args=(r, 2, uid, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r = q.get(timeout=300)
        res[r[0]] = r[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rows0, plan0 = np.array(res[0][0]), res[0][1]
    assert np.array_equal(rows0, np.array(res[1][0])) and plan0 == res[1][1]
    # every request was observed in every slot (non-binding capacities: no idling)
    assert np.all(rows0[..., 1].sum(-1) == SLOTS)
    for r in (0, 1):
        tokens, served, committed, plens = res[r][2], res[r][3], res[r][4], res[r][5]
        assert served == SLOTS * len(committed)
        assert tokens == sum(c - p for c, p in zip(committed, plens))  # accepted + bonus = committed growth
