"""Request-level data parallelism -- a thin Python view of
the C-ABI communicator in libspin.so (csrc/comm.cpp, spin_comm_* in
include/spin_c.h).

Requests are sharded in contiguous blocks across ranks (weights replicated); the
only exchange is an all-gather of per-(request, SSM) acceptance statistics (the
reference's ArmEstimate{sum, count}, bandit.hpp:24-39). All-gather (not
all-reduce) keeps the host reduction order fixed (rank order), so every rank
derives identical selector inputs. Backends: NCCL (GPUs) and TCP (same
semantics without a GPU; the CPU tests).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib

NCCL, TCP = 0, 1
SUM, MAX = 0, 1


def shard(num_requests: int, world: int, rank: int) -> range:
    """Contiguous block of request ids owned by `rank` (sizes differ by <= 1)."""
    base, extra = divmod(num_requests, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def unique_id(backend: int) -> bytes:
    buf = (C.c_uint8 * 128)()
    _lib.check(_lib.load().spin_comm_unique_id(backend, buf))
    return bytes(buf)


class Comm:
    """One communicator per process / device (spin_comm)."""

    def __init__(self, backend: int, rank: int, world: int, uid: bytes, device: int = 0):
        self.lib = _lib.load()
        self.rank, self.world, self.backend = rank, world, backend
        buf = (C.c_uint8 * 128).from_buffer_copy(uid.ljust(128, b"\0"))
        h = C.c_void_p()
        _lib.check(self.lib.spin_comm_create(backend, device, rank, world, buf, C.byref(h)))
        self.h = h

    @classmethod
    def from_env(cls, backend: int = NCCL, device: int | None = None) -> "Comm":
        """Rank / world from RANK / WORLD_SIZE; the id from SPIN_COMM_ID (hex), which the
        launcher (bench.py) creates once and hands to every rank."""
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        uid = bytes.fromhex(os.environ["SPIN_COMM_ID"])
        dev = int(os.environ.get("LOCAL_RANK", "0")) if device is None else device
        return cls(backend, rank, world, uid, dev)

    def close(self):
        if self.h:
            _lib.check(self.lib.spin_comm_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def allreduce(self, values, op: int = SUM) -> np.ndarray:
        v = np.ascontiguousarray(values, dtype=np.float64).copy()
        _lib.check(self.lib.spin_comm_allreduce(self.h, v.ctypes.data_as(_lib.P_F64), v.size, op))
        return v

    def max(self, x: float) -> float:
        return float(self.allreduce([x], MAX)[0])

    def sum(self, x: float) -> float:
        return float(self.allreduce([x], SUM)[0])

    def barrier(self) -> None:
        _lib.check(self.lib.spin_comm_barrier(self.h))


class AcceptanceStats:
    """Local ArmEstimate rows [rows, n_ssm, (sum, count)] (host) plus the gather."""

    def __init__(self, num_requests: int, n_ssm: int, world: int, rank: int):
        self.world, self.rank, self.n_ssm = world, rank, n_ssm
        self.num_requests = num_requests
        self.owned = shard(num_requests, world, rank)
        self.rows = max(len(shard(num_requests, world, r)) for r in range(world))  # padded for the gather
        self.host = np.zeros((self.rows, n_ssm, 2), np.float64)

    def add(self, local_index: int, ssm: int, goodput: float) -> None:
        """ArmEstimate::add (bandit.hpp:28-31)."""
        self.host[local_index, ssm, 0] += goodput
        self.host[local_index, ssm, 1] += 1

    def add_many(self, local_indices, ssms, goodputs) -> None:
        """ArmEstimate::add for a batch of (request, SSM, goodput) observations, in order."""
        np.add.at(self.host[..., 0], (np.asarray(local_indices), np.asarray(ssms)), np.asarray(goodputs, np.float64))
        np.add.at(self.host[..., 1], (np.asarray(local_indices), np.asarray(ssms)), 1.0)

    def gather(self, comm: Comm | None = None) -> np.ndarray:
        """spin_stats_allgather; returns global [num_requests, n_ssm, 2] in request-id order."""
        if comm is None or self.world == 1:
            return self.host[: len(self.owned)].copy()
        out = np.zeros((self.world * self.rows, self.n_ssm, 2), np.float64)
        _lib.check(comm.lib.spin_stats_allgather(comm.h, self.host.ctypes.data_as(_lib.P_F64),
                                                 out.ctypes.data_as(_lib.P_F64), self.rows, self.n_ssm))
        parts = [out[r * self.rows: r * self.rows + len(shard(self.num_requests, self.world, r))]
                 for r in range(self.world)]
        return np.concatenate(parts, 0)

    @staticmethod
    def means(global_rows: np.ndarray) -> np.ndarray:
        """Per-(request, SSM) mean goodput; +inf where unobserved (optimistic_mean, bandit.hpp:36-38)."""
        s, c = global_rows[..., 0], global_rows[..., 1]
        with np.errstate(invalid="ignore", divide="ignore"):
            return np.where(c > 0, s / np.maximum(c, 1), np.inf)
