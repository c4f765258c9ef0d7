"""The device request decomposition the hot path runs (meta_kernel's warp packer,
kernels.cu) is bit-identical to the reference packer (packing.cpp:16-103) on
every golden case, and to the host packer on large random batches."""
import ctypes as C

import numpy as np
import pytest

from paper_2503_15921_b200 import _lib
from tests._golden import golden

pytestmark = pytest.mark.gpu


def pack(fn, lens, width):
    n = len(lens)
    cap = 2 * n + 4
    kv = np.array(lens or [0], dtype=np.int32)
    segs = (_lib.Segment * cap)()
    reps = np.zeros(max(n, 1), dtype=np.int32)
    L, rows, ns = C.c_int32(), C.c_int32(), C.c_int32()
    pad = C.c_int64()
    st = fn(kv.ctypes.data_as(_lib.P_I32), n, width, C.byref(L), C.byref(rows), segs, cap, C.byref(ns), C.byref(pad),
            reps.ctypes.data_as(_lib.P_I32))
    seg_list = [[s.request_id, s.row, s.col_start, s.col_end, s.token_offset] for s in segs[: ns.value]]
    return st, L.value, rows.value, pad.value, seg_list, reps[:n].tolist()


def test_device_packer_matches_reference_goldens():
    lib = _lib.load()
    cases = golden()["pack"]
    checked = 0
    for case in cases:
        st, L, rows, pad, segs, reps = pack(lib.spin_pack_device, case["lens"], case["width"])
        assert st == case["status"], (case, lib.spin_last_error())
        if st == 0:
            assert (L, rows, pad, segs, reps) == (case["length"], case["rows"], case["padding"], case["segments"],
                                                  case["q_replica_rows"]), case
            checked += 1
    assert checked >= 300


@pytest.mark.parametrize("n,width,lo,hi", [(32, 32, 128, 600), (64, 8, 1, 2000), (256, 64, 100, 520),
                                           (1024, 1024, 1, 700), (1000, 37, 1, 50), (97, 5, 1, 4)])
def test_device_packer_matches_host_packer_at_scale(n, width, lo, hi):
    lib = _lib.load()
    rng = np.random.default_rng(n * 7 + width)
    for _ in range(5):
        lens = rng.integers(lo, hi + 1, n).tolist()
        assert pack(lib.spin_pack_device, lens, width) == pack(lib.spin_pack, lens, width)


def test_device_packer_rejects_oversize_batch():
    st = pack(_lib.load().spin_pack_device, [3] * 1025, 4)[0]
    assert _lib.STATUS_NAMES[st] == "SizeError"
