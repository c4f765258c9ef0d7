"""Learning-based SSM selection (LBSS) on measured goodput -- a thin Python view of
the C++ selector in libspin.so (csrc/lbss.cpp; C ABI spin_lbss_* in
include/spin_c.h), which restates the reference's bandit (proj/core/src/bandit.cpp,
include/specsim/bandit.hpp, src/matching.cpp) with the same draw order, schedule and
tie-breaking. No selection logic lives here.

Epoch k (bandit.cpp:248-332): an exploration stage of `alpha` slots in chunks of
`beta` slots, each chunk with a fresh random request -> SSM draw that respects the
per-SSM capacities (draw_exploration_assignment / resolve_capacity_overflow,
bandit.cpp:61-120); then an exploitation stage of 2^k slots (exploitation_duration,
bandit.cpp:54-59) on the max-weight matching of the per-(request, SSM) goodput
estimates (plan_exploitation, bandit.cpp:186-226). Every slot adds
observed_goodput = (accepted + bonus) / wall seconds (model.cpp:165-171) to the
served arm (ArmEstimate::add, bandit.hpp:28-31).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


class Lbss:
    def __init__(self, num_requests: int, capacities, alpha: int = 8, beta: int = 2, seed: int = 2503):
        self.lib = _lib.load()
        self.n, self.m = int(num_requests), len(capacities)
        caps = np.ascontiguousarray(capacities, dtype=np.int32)
        h = C.c_void_p()
        _lib.check(self.lib.spin_lbss_create(self.n, self.m, caps.ctypes.data_as(_lib.P_I32), alpha, beta, seed,
                                             C.byref(h)))
        self.h = h
        self.epoch = 1
        self.prewarm = np.full(self.n, -1, np.int32)

    def close(self):
        if self.h:
            _lib.check(self.lib.spin_lbss_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def next_slot(self):
        """(assignment [n] -> ssm or -1, explore flag); self.prewarm / self.epoch follow."""
        a = np.zeros(self.n, np.int32)
        ex, ep = C.c_int32(), C.c_int32()
        _lib.check(self.lib.spin_lbss_next(self.h, a.ctypes.data_as(_lib.P_I32), self.prewarm.ctypes.data_as(_lib.P_I32),
                                           C.byref(ex), C.byref(ep)))
        self.epoch = ep.value
        return a, bool(ex.value)

    def add(self, request: int, ssm: int, goodput: float) -> None:
        _lib.check(self.lib.spin_lbss_observe(self.h, int(request), int(ssm), float(goodput)))

    def exploitation(self) -> np.ndarray:
        """plan_exploitation on the current estimates."""
        a = np.zeros(self.n, np.int32)
        _lib.check(self.lib.spin_lbss_plan(self.h, a.ctypes.data_as(_lib.P_I32)))
        return a

    def rows(self) -> np.ndarray:
        r = np.zeros((self.n, self.m, 2), np.float64)
        _lib.check(self.lib.spin_lbss_rows(self.h, r.ctypes.data_as(_lib.P_F64), 0))
        return r

    def set_rows(self, rows) -> None:
        r = np.ascontiguousarray(rows, dtype=np.float64)
        assert r.shape == (self.n, self.m, 2)
        _lib.check(self.lib.spin_lbss_rows(self.h, r.ctypes.data_as(_lib.P_F64), 1))
