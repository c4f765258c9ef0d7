"""The NCCL transport of the C-ABI communicator on a real GPU (spin_comm_*: libnccl loaded
with dlopen, one communicator per device): a world-1 communicator all-gathers per-(request,
SSM) ArmEstimate rows through spin_stats_allgather and reduces scalars -- the code path
`bench.py --gpus N` takes on every rank of an N-GPU node (N > 1 needs one GPU per rank; every
lease here has one)."""
import numpy as np
import pytest

from paper_2503_15921_b200 import _lib, dist
from paper_2503_15921_b200.dist import NCCL, Comm

pytestmark = pytest.mark.gpu


def test_nccl_world1_allgather_and_reductions():
    comm = Comm(NCCL, 0, 1, dist.unique_id(NCCL), device=0)
    rows, n_ssm = 6, 3
    local = np.zeros((rows, n_ssm, 2), np.float64)
    for i in range(rows):
        local[i, i % n_ssm] = (20.0 * i + 4.0, 2.0)
    out = np.full_like(local, -1.0)
    _lib.check(comm.lib.spin_stats_allgather(comm.h, local.ctypes.data_as(_lib.P_F64), out.ctypes.data_as(_lib.P_F64),
                                             rows, n_ssm))
    assert np.array_equal(out, local)
    assert comm.max(3.5) == 3.5 and comm.sum(2.25) == 2.25
    comm.close()
