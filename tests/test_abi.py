"""The C-ABI library loads, exports every symbol include/spin_c.h declares,
and its host-side entry points (no GPU needed) match the reference goldens."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2503_15921_b200 import _lib
from tests._golden import golden

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def header_symbols():
    text = open(os.path.join(ROOT, "include", "spin_c.h")).read()
    return sorted(set(re.findall(r"^\s*(?:spin_status|int|const char\*)\s+(spin_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, f"declared in spin_c.h but not exported: {missing}"
    assert set(syms) <= set(_lib.exported_symbols())
    assert lib.spin_abi_version() == 3


def spin_pack(lens, width):
    lib = _lib.load()
    n = len(lens)
    cap = 2 * n + 4
    kv = np.array(lens or [0], dtype=np.int32)
    segs = (_lib.Segment * cap)()
    reps = np.zeros(max(n, 1), dtype=np.int32)
    L, rows, ns = C.c_int32(), C.c_int32(), C.c_int32()
    pad = C.c_int64()
    st = lib.spin_pack(kv.ctypes.data_as(_lib.P_I32), n, width, C.byref(L), C.byref(rows), segs, cap, C.byref(ns),
                       C.byref(pad), reps.ctypes.data_as(_lib.P_I32))
    seg_list = [[s.request_id, s.row, s.col_start, s.col_end, s.token_offset] for s in segs[: ns.value]]
    return st, L.value, rows.value, pad.value, seg_list, reps[:n].tolist()


def test_spin_pack_bit_identical_to_reference():
    for case in golden()["pack"]:
        st, L, rows, pad, segs, reps = spin_pack(case["lens"], case["width"])
        assert st == case["status"], (case, _lib.load().spin_last_error())
        if st == 0:
            assert (L, rows, pad, segs, reps) == (case["length"], case["rows"], case["padding"], case["segments"],
                                                  case["q_replica_rows"])


def test_spin_pack_error_mapping():
    lib = _lib.load()
    st = spin_pack([1, 2], 0)[0]
    assert _lib.STATUS_NAMES[st] == "ConfigError"
    assert b"width" in lib.spin_last_error()
    with pytest.raises(_lib.SpinError) as ei:
        _lib.check(spin_pack([0], 2)[0])
    assert ei.value.kind == "ConfigError"


def test_spin_verify_cost_and_naive_padding_match_reference():
    lib = _lib.load()
    for case in golden()["verify_batch_cost"]:
        kv = np.array(case["lens"], dtype=np.int32)
        tok, pad = C.c_int64(), C.c_int64()
        st = lib.spin_verify_batch_cost(kv.ctypes.data_as(_lib.P_I32), len(case["lens"]), case["window"],
                                        case["packing"], case["width"], C.byref(tok), C.byref(pad))
        assert st == case["status"] and (tok.value, pad.value) == (case["tokens"], case["padding"])
    for case in golden()["naive_padding"]:
        kv = np.array(case["lens"] or [0], dtype=np.int32)
        pad = C.c_int64()
        st = lib.spin_naive_padding(kv.ctypes.data_as(_lib.P_I32), len(case["lens"]), C.byref(pad))
        assert st == case["status"]
        if st == 0:
            assert pad.value == case["padding"]
