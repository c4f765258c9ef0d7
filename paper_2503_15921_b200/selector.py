"""Learning-based SSM selection (LBSS) on measured goodput -- the host selector of
Spin, restated from the reference's bandit (reference: proj/core/src/bandit.cpp,
include/specsim/bandit.hpp) to drive the B200 engine from Python (bench config c4).
The C++ drop-in (oracle/dropin/lbss_on_b200.cpp) runs the reference's own
unmodified bandit.cpp against the same engine through include/specsim.

Epoch k (bandit.cpp:248-332): an exploration stage of `alpha` slots in chunks of
`beta` slots, each chunk with a fresh uniformly random request -> SSM draw that
respects per-SSM capacities (draw_exploration_assignment / resolve_capacity_overflow,
bandit.cpp:61-120); then an exploitation stage of 2^k slots (exploitation_duration,
bandit.cpp:54-59) on the max-weight matching of the per-(request, SSM) goodput
estimates under the capacities (plan_exploitation, bandit.cpp:186-226), unobserved
arms clamped to one above the best finite estimate. Every slot adds
observed_goodput = (accepted + bonus) / slot seconds (model.cpp:165-171) to the
served arm (ArmEstimate::add, bandit.hpp:28-31).
"""
from __future__ import annotations

import numpy as np


class Lbss:
    def __init__(self, num_requests: int, capacities, alpha: int = 8, beta: int = 2, seed: int = 2503):
        if alpha < 1 or beta < 1 or alpha % beta != 0:
            raise ValueError("LBSS: beta must divide alpha")  # validate(BanditConfig), bandit.cpp:11-23
        self.n = num_requests
        self.cap = np.asarray(capacities, dtype=np.int64)
        self.m = len(self.cap)
        self.alpha, self.beta = alpha, beta
        self.rng = np.random.default_rng(seed)
        self.sum = np.zeros((self.n, self.m))
        self.count = np.zeros((self.n, self.m), dtype=np.int64)
        self.epoch = 1
        self._plan = self._iter()

    # ---- estimates (ArmEstimate)
    def add(self, request: int, ssm: int, goodput: float) -> None:
        self.sum[request, ssm] += goodput
        self.count[request, ssm] += 1

    def means(self) -> np.ndarray:
        with np.errstate(invalid="ignore", divide="ignore"):
            return np.where(self.count > 0, self.sum / np.maximum(self.count, 1), np.inf)

    # ---- assignments
    def _resolve_capacity(self, desired: np.ndarray) -> np.ndarray:
        """resolve_capacity_overflow (bandit.cpp:61-106): keep a random subset per SSM up to
        its capacity; overflow requests go to a random SSM with room, else idle (-1)."""
        res = desired.copy()
        load = np.zeros(self.m, dtype=np.int64)
        overflow = []
        for j in range(self.m):
            members = np.flatnonzero(res == j)
            if len(members) <= self.cap[j]:
                load[j] = len(members)
                continue
            self.rng.shuffle(members)
            load[j] = self.cap[j]
            overflow.extend(members[self.cap[j]:].tolist())
        for rid in sorted(overflow):
            open_ = np.flatnonzero(load < self.cap)
            if len(open_) == 0:
                res[rid] = -1
                continue
            j = int(self.rng.choice(open_))
            res[rid] = j
            load[j] += 1
        return res

    def exploration(self) -> np.ndarray:
        return self._resolve_capacity(self.rng.integers(0, self.m, self.n))

    def exploitation(self) -> np.ndarray:
        """Max-weight matching of requests to SSM capacity replicas (plan_exploitation)."""
        mu = self.means()
        finite = mu[np.isfinite(mu)]
        cold = (finite.max() + 1.0) if finite.size else 1.0
        w = np.where(np.isfinite(mu), mu, cold)
        if np.all(self.cap >= self.n):  # capacities do not bind: per-request argmax (lowest id on ties)
            return np.argmax(w, axis=1).astype(np.int64)
        from scipy.optimize import linear_sum_assignment

        cols = np.concatenate([np.full(int(min(c, self.n)), j) for j, c in enumerate(self.cap)])
        rows, picks = linear_sum_assignment(-w[:, cols])
        out = np.full(self.n, -1, dtype=np.int64)
        out[rows] = cols[picks]
        return out

    def _iter(self):
        while True:
            for _ in range(self.alpha // self.beta):  # exploration chunks
                a = self.exploration()
                for _ in range(self.beta):
                    yield a, True
            plan = self.exploitation()
            for _ in range(2 ** min(self.epoch, 30)):  # exploitation_duration
                yield plan, False
            self.epoch += 1

    def next_slot(self):
        """(assignment [n] -> ssm or -1, explore flag) for the next slot."""
        return next(self._plan)
