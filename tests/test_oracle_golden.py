"""Pins the CPU oracle (oracle/, plain-C restatement) against golden vectors
produced by the UNMODIFIED reference (oracle/make_golden.py) and, when the
reference build is present, against the reference library directly."""
import ctypes as C

import numpy as np
import pytest

from oracle import load_oracle
from tests._golden import golden


def ptr(a):
    return a.ctypes.data_as(C.c_void_p)


@pytest.fixture(scope="module")
def so():
    return load_oracle()


def test_rng_matches_reference(so):
    for case in golden()["rng"]:
        r = (C.c_uint64 * 313)()
        so.so_rng_init(r, case["seed"])
        assert [so.so_rng_next(r) for _ in range(16)] == case["next"]
        so.so_rng_init(r, case["seed"])
        assert [so.so_rng_unit(r) for _ in range(16)] == case["unit"]
        so.so_rng_init(r, case["seed"])
        assert [so.so_rng_uniform_int(r, 1, 6) for _ in range(16)] == case["uniform_int_1_6"]
        assert so.so_mix_seed(case["seed"], 3, 7, 11) == case["mix_seed"]


def test_toy_inputs_match_reference(so):
    for case in golden()["toy_inputs"]:
        q = np.zeros(case["queries"] * case["dim"])
        k = np.zeros(case["kv_len"] * case["dim"])
        v = np.zeros(case["kv_len"] * case["dim"])
        so.so_make_toy_input(case["seed"], case["queries"], case["kv_len"], case["dim"], ptr(q), ptr(k), ptr(v))
        assert q.tolist() == case["q"] and k.tolist() == case["k"] and v.tolist() == case["v"]


def oracle_pack(so, lens, width):
    n = len(lens)
    cap = 2 * n + 4
    kv = np.array(lens or [0], dtype=np.int32)
    segs = np.zeros(5 * cap, dtype=np.int32)
    reps = np.zeros(max(n, 1), dtype=np.int32)
    L, rows, ns = C.c_int(), C.c_int(), C.c_int()
    pad = C.c_longlong()
    st = so.so_pack(ptr(kv), n, width, C.byref(L), C.byref(rows), ptr(segs), cap, C.byref(ns), C.byref(pad),
                    ptr(reps))
    return st, L.value, rows.value, pad.value, segs[: 5 * ns.value].reshape(-1, 5).tolist(), reps[:n].tolist()


def test_pack_matches_reference(so):
    for case in golden()["pack"]:
        st, L, rows, pad, segs, reps = oracle_pack(so, case["lens"], case["width"])
        assert st == case["status"], case
        if st == 0:
            assert (L, rows, pad) == (case["length"], case["rows"], case["padding"]), case
            assert segs == case["segments"]
            assert reps == case["q_replica_rows"]


def test_reference_packing_known_answers(so):
    # test_packing.cpp:38-87
    assert oracle_pack(so, [4, 4, 4], 3)[1:4] == (4, 3, 0)
    st, L, rows, pad, segs, reps = oracle_pack(so, [8, 5, 3], 2)
    assert (L, pad) == (8, 0)
    st, L, rows, pad, segs, reps = oracle_pack(so, [10, 2], 2)
    assert (L, pad, reps) == (6, 0, [2, 1])


def test_naive_padding_and_verify_cost(so):
    for case in golden()["naive_padding"]:
        pad = C.c_longlong()
        kv = np.array(case["lens"] or [0], dtype=np.int32)
        assert so.so_naive_padding(ptr(kv), len(case["lens"]), C.byref(pad)) == case["status"]
        if case["status"] == 0:
            assert pad.value == case["padding"]
    for case in golden()["verify_batch_cost"]:
        kv = np.array(case["lens"], dtype=np.int32)
        tok, pad = C.c_longlong(), C.c_longlong()
        st = so.so_verify_batch_cost(ptr(kv), len(case["lens"]), case["window"], case["packing"], case["width"],
                                     C.byref(tok), C.byref(pad))
        assert st == case["status"]
        assert (tok.value, pad.value) == (case["tokens"], case["padding"])


def test_attention_matches_reference(so):
    for case in golden()["attention"]:
        dim = case["dim"]
        qs, ks, vs, qr, kr = [], [], [], [], []
        for seed, q, kv in case["specs"]:
            Q, K, V = np.zeros(q * dim), np.zeros(kv * dim), np.zeros(kv * dim)
            so.so_make_toy_input(seed, q, kv, dim, ptr(Q), ptr(K), ptr(V))
            qs.append(Q), ks.append(K), vs.append(V), qr.append(q), kr.append(kv)
        Q, K, V = np.concatenate(qs), np.concatenate(ks), np.concatenate(vs)
        st, L, rows, pad, segs, reps = oracle_pack(so, kr, case["width"])
        segs_a = np.array(segs, dtype=np.int32).ravel()
        out = np.zeros(Q.size)
        qr_a, kr_a = np.array(qr, dtype=np.int32), np.array(kr, dtype=np.int32)
        st = so.so_decomposed_attention(len(qr), dim, ptr(qr_a), ptr(kr_a), ptr(Q), ptr(K), ptr(V), ptr(segs_a),
                                        len(segs), rows, L, None, ptr(out))
        assert st == case["status"] == 0
        # the restatement follows the reference loop order: identical doubles
        assert out.tolist() == case["decomposed"]
        ref = np.array(case["reference"])
        assert np.abs(out - ref).max() <= 1e-9  # acceptance.cpp:72-101 / test_attention.cpp:94-161
        qo = ko = 0
        for q, kv in zip(qr, kr):
            o = np.zeros(q * dim)
            assert so.so_reference_attention(q, kv, dim, ptr(Q[qo * dim:]), ptr(K[ko * dim:]), ptr(V[ko * dim:]),
                                             ptr(o)) == 0
            assert o.tolist() == case["reference"][qo * dim:(qo + q) * dim]
            qo += q
            ko += kv


def test_decomposed_attention_rejects_bad_layouts(so):
    # test_attention.cpp:124-138
    dim = 4
    Q, K, V = np.zeros(2 * dim), np.zeros(5 * dim), np.zeros(5 * dim)
    so.so_make_toy_input(51, 2, 5, dim, ptr(Q), ptr(K), ptr(V))
    st, L, rows, pad, segs, reps = oracle_pack(so, [4], 1)  # one token short
    out = np.zeros(Q.size)
    qr, kr = np.array([2], dtype=np.int32), np.array([5], dtype=np.int32)
    segs_a = np.array(segs, dtype=np.int32).ravel()
    assert so.so_decomposed_attention(1, dim, ptr(qr), ptr(kr), ptr(Q), ptr(K), ptr(V), ptr(segs_a), len(segs), rows,
                                      L, None, ptr(out)) == 5


def test_acceptance_semantics(so):
    for case in golden()["acceptance"]:
        r = (C.c_uint64 * 313)()
        so.so_rng_init(r, case["seed"])
        draws = [so.so_sample_accepted_prefix(case["p"], case["window"], r) for _ in range(64)]
        assert draws == case["draws"]
        assert so.so_expected_accepted_prefix(case["p"], case["window"]) == case["expected"]
    assert abs(so.so_expected_accepted_prefix(0.8, 4) - 2.3616) < 1e-12  # test_model.cpp:112-142
