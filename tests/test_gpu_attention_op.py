"""spin_decomposed_attention (GPU, fp64, split-KV + shared-max combine) against
the reference's decomposed_attention / reference_attention golden outputs."""
import ctypes as C

import numpy as np
import pytest

from oracle import load_oracle
from paper_2503_15921_b200 import _lib
from tests._golden import golden

pytestmark = pytest.mark.gpu


def ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def host_pack(lens, width):
    n = len(lens)
    cap = 2 * n + 4
    kv = np.array(lens, dtype=np.int32)
    segs = (_lib.Segment * cap)()
    reps = np.zeros(n, dtype=np.int32)
    L, rows, ns = C.c_int32(), C.c_int32(), C.c_int32()
    pad = C.c_int64()
    _lib.check(_lib.load().spin_pack(ptr(kv, C.c_int32), n, width, C.byref(L), C.byref(rows), segs, cap, C.byref(ns),
                                     C.byref(pad), ptr(reps, C.c_int32)))
    return segs, ns.value, rows.value, L.value


def test_decomposed_attention_matches_reference_goldens():
    lib = _lib.load()
    so = load_oracle()
    worst = 0.0
    for case in golden()["attention"]:
        dim = case["dim"]
        qs, ks, vs, qr, kr = [], [], [], [], []
        for seed, q, kv in case["specs"]:
            Q, K, V = np.zeros(q * dim), np.zeros(kv * dim), np.zeros(kv * dim)
            so.so_make_toy_input(seed, q, kv, dim, Q.ctypes.data, K.ctypes.data, V.ctypes.data)
            qs.append(Q), ks.append(K), vs.append(V), qr.append(q), kr.append(kv)
        Q, K, V = np.concatenate(qs), np.concatenate(ks), np.concatenate(vs)
        segs, ns, rows, L = host_pack(kr, case["width"])
        out = np.zeros(Q.size)
        qr_a, kr_a = np.array(qr, np.int32), np.array(kr, np.int32)
        _lib.check(lib.spin_decomposed_attention(len(qr), dim, ptr(qr_a, C.c_int32), ptr(kr_a, C.c_int32),
                                                 ptr(Q, C.c_double), ptr(K, C.c_double), ptr(V, C.c_double), segs, ns,
                                                 rows, L, None, ptr(out, C.c_double)))
        ref = np.array(case["reference"])
        worst = max(worst, float(np.abs(out - ref).max()))
        assert np.abs(out - np.array(case["decomposed"])).max() <= 1e-12
    assert worst <= 1e-12, worst


def test_decomposed_attention_rejects_inconsistent_layout():
    lib = _lib.load()
    dim = 4
    Q, K, V = np.zeros(2 * dim), np.zeros(5 * dim), np.zeros(5 * dim)
    segs, ns, rows, L = host_pack([4], 1)  # one token short (test_attention.cpp:133-138)
    out = np.zeros(Q.size)
    qr, kr = np.array([2], np.int32), np.array([5], np.int32)
    st = lib.spin_decomposed_attention(1, dim, ptr(qr, C.c_int32), ptr(kr, C.c_int32), ptr(Q, C.c_double),
                                       ptr(K, C.c_double), ptr(V, C.c_double), segs, ns, rows, L, None,
                                       ptr(out, C.c_double))
    assert _lib.STATUS_NAMES[st] == "ConsistencyError"
