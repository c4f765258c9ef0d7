"""Request-level data parallelism.

Requests are sharded in contiguous blocks across ranks (weights replicated);
the only exchange is an all-gather of per-(request, SSM) acceptance statistics
(the reference's ArmEstimate{sum, count}, bandit.hpp:24-39). All-gather (not
all-reduce) keeps the host reduction order fixed (rank order), so every rank
derives identical selector inputs. Backend-agnostic: NCCL on GPUs, gloo in the
CPU tests.
"""
from __future__ import annotations

import numpy as np
import torch


def shard(num_requests: int, world: int, rank: int) -> range:
    """Contiguous block of request ids owned by `rank` (sizes differ by <= 1)."""
    base, extra = divmod(num_requests, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


class AcceptanceStats:
    """Local ArmEstimate rows [local_requests, n_ssm, (sum, count)] plus the gather.

    The rows are accumulated on the host (a numpy view of a CPU tensor: per-request
    updates are host arithmetic, not device launches); `device` holds the gather
    buffers (CUDA for NCCL), filled by one host->device copy per gather."""

    def __init__(self, num_requests: int, n_ssm: int, world: int, rank: int, device="cpu"):
        self.world, self.rank = world, rank
        self.owned = shard(num_requests, world, rank)
        self.rows = max(len(shard(num_requests, world, r)) for r in range(world))  # padded for the gather
        self.host = torch.zeros((self.rows, n_ssm, 2), dtype=torch.float64)
        self._np = self.host.numpy()
        self.local = torch.zeros((self.rows, n_ssm, 2), dtype=torch.float64, device=device)
        # flat [world * rows, ...]: the layout all_gather_into_tensor fills (gloo and NCCL)
        self.gathered = torch.zeros((world * self.rows, n_ssm, 2), dtype=torch.float64, device=device)
        self.num_requests = num_requests

    def add(self, local_index: int, ssm: int, goodput: float) -> None:
        """ArmEstimate::add (bandit.hpp:28-31)."""
        self._np[local_index, ssm, 0] += goodput
        self._np[local_index, ssm, 1] += 1

    def add_many(self, local_indices, ssms, goodputs) -> None:
        """ArmEstimate::add for a batch of (request, SSM, goodput) observations, in order."""
        np.add.at(self._np[..., 0], (np.asarray(local_indices), np.asarray(ssms)), np.asarray(goodputs, np.float64))
        np.add.at(self._np[..., 1], (np.asarray(local_indices), np.asarray(ssms)), 1.0)

    def gather(self, dist=None) -> torch.Tensor:
        """All-gather; returns global [num_requests, n_ssm, 2] in request-id order."""
        if dist is not None and self.world > 1:
            self.local.copy_(self.host)
            dist.all_gather_into_tensor(self.gathered, self.local)
            parts = [self.gathered[r * self.rows: r * self.rows + len(shard(self.num_requests, self.world, r))]
                     for r in range(self.world)]
            return torch.cat(parts, 0)
        return self.host[: len(self.owned)].clone()

    @staticmethod
    def means(global_rows: torch.Tensor) -> torch.Tensor:
        """Per-(request, SSM) mean goodput; +inf where unobserved (optimistic_mean, bandit.hpp:36-38)."""
        s, c = global_rows[..., 0], global_rows[..., 1]
        return torch.where(c > 0, s / c.clamp_min(1), torch.full_like(s, float("inf")))
