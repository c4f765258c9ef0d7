"""Generates tests/golden/reference_golden.json by running the UNMODIFIED
reference functions (oracle/_ref/libspecsim_ref.so, compiled from
/root/reference/proj/core sources by `make -C oracle ref`).

Run here (where /root/reference exists):  python oracle/make_golden.py
The JSON is committed; the GPU box never reads /root/reference.

Cases follow the reference's own tests:
  rng / mix_seed        rng.hpp:11-68
  make_toy_input        attention.cpp:164-175
  pack / naive_padding  test_packing.cpp:38-169 (+ random trials, seeds 99/313/808)
  verify_batch_cost     slot_engine.cpp:24-45
  attention             test_attention.cpp:85-161 (seeds 21, 22/23, 31-33, random 424242)
  acceptance            test_model.cpp:112-142 (p = 0, 0.8, 1; E = 2.3616)

`python oracle/make_golden.py toy_bf16` writes tests/golden/toy_bf16_golden.json: the
reference's reference_attention and decomposed_attention (pack width as given) on
make_toy_input data whose K / V are rounded to bf16 and Q to fp32 -- the operand
precisions of the production attention kernel -- so that kernel, run in toy mode
(scale 1, non-causal), can be pinned to the reference's own outputs.

`python oracle/make_golden.py lbss` writes tests/golden/lbss_golden.json: the
reference selector's assignment / prewarm / explore trace (run_lbss control flow,
bandit.cpp:248-332, replayed by ref_lbss_trace in oracle/ref_shim.cpp) on seeded
synthetic goodput tables, binding and non-binding capacities.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import load_ref  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "reference_golden.json")


def ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def ref_pack(lib, lens, width):
    n = len(lens)
    cap = 2 * n + 4
    kv = np.array(lens, dtype=np.int32)
    segs = np.zeros(5 * cap, dtype=np.int32)
    reps = np.zeros(max(n, 1), dtype=np.int32)
    L, rows, ns = C.c_int(), C.c_int(), C.c_int()
    pad = C.c_longlong()
    st = lib.ref_pack(ptr(kv), n, width, C.byref(L), C.byref(rows), ptr(segs), cap, C.byref(ns), C.byref(pad),
                      ptr(reps))
    if st:
        return {"lens": lens, "width": width, "status": st}
    return {"lens": lens, "width": width, "status": 0, "length": L.value, "rows": rows.value,
            "padding": pad.value, "segments": segs[: 5 * ns.value].reshape(-1, 5).tolist(),
            "q_replica_rows": reps[:n].tolist()}


def main():
    lib = load_ref()
    rng = np.random.default_rng(2503)
    g = {}
    # ---- rng
    rr = []
    for seed in [0, 1, 2503, 424242, 2**63 + 11]:
        u = np.zeros(16, dtype=np.uint64)
        d = np.zeros(16, dtype=np.float64)
        lib.ref_rng_draws(seed, 0, 0, 0, 16, ptr(d), ptr(u))
        nxt = [int(x) for x in u]
        lib.ref_rng_draws(seed, 1, 0, 0, 16, ptr(d), ptr(u))
        unit = d.tolist()
        lib.ref_rng_draws(seed, 2, 1, 6, 16, ptr(d), ptr(u))
        ui = [int(x) for x in u]
        rr.append({"seed": seed, "next": nxt, "unit": unit, "uniform_int_1_6": ui,
                   "mix_seed": int(lib.ref_mix_seed(seed, 3, 7, 11))})
    g["rng"] = rr
    # ---- toy inputs
    toys = []
    for seed, q, kv, dim in [(7, 3, 1, 4), (21, 3, 6, 4), (1000, 3, 8, 4), (5, 2, 3, 8)]:
        Q = np.zeros(q * dim)
        K = np.zeros(kv * dim)
        V = np.zeros(kv * dim)
        lib.ref_make_toy_input(seed, q, kv, dim, ptr(Q), ptr(K), ptr(V))
        toys.append({"seed": seed, "queries": q, "kv_len": kv, "dim": dim, "q": Q.tolist(), "k": K.tolist(),
                     "v": V.tolist()})
    g["toy_inputs"] = toys
    # ---- pack
    cases = [([4, 4, 4], 3), ([8, 5, 3], 2), ([7, 5, 5], 3), ([10, 2], 2), ([5], 1), ([5, 3], 2), ([1, 2], 0),
             ([0], 2), ([], 3), ([100], 7), ([3, 3, 3, 3, 3], 2)]
    for _ in range(300):
        n = int(rng.integers(1, 11))
        cases.append(([int(x) for x in rng.integers(1, 41, n)], int(rng.integers(1, 7))))
    for _ in range(20):  # verify-sized batches: prompt U[128,512] + generated + gamma
        n = int(rng.choice([8, 32, 64]))
        cases.append(([int(x) for x in rng.integers(128, 600, n)], n))
    g["pack"] = [ref_pack(lib, lens, w) for lens, w in cases]
    # ---- naive padding + verify cost
    np_cases = []
    for lens in [[4, 4, 4], [7, 5, 5], [8, 5, 3], []]:
        kv = np.array(lens or [0], dtype=np.int32)
        pad = C.c_longlong()
        st = lib.ref_naive_padding(ptr(kv), len(lens), C.byref(pad))
        np_cases.append({"lens": lens, "status": st, "padding": pad.value})
    g["naive_padding"] = np_cases
    vc = []
    for _ in range(60):
        n = int(rng.integers(1, 40))
        lens = [int(x) for x in rng.integers(1, 600, n)]
        window = int(rng.integers(1, 17))
        packing = int(rng.integers(0, 2))
        width = int(rng.integers(0, n + 2))
        kv = np.array(lens, dtype=np.int32)
        tok, pad = C.c_longlong(), C.c_longlong()
        st = lib.ref_verify_batch_cost(ptr(kv), n, window, packing, width, C.byref(tok), C.byref(pad))
        vc.append({"lens": lens, "window": window, "packing": packing, "width": width, "status": st,
                   "tokens": tok.value, "padding": pad.value})
    g["verify_batch_cost"] = vc
    # ---- attention (toy mode)
    att = []

    def att_case(specs, width, dim=4):
        qs, ks, vs, qr, kr = [], [], [], [], []
        for seed, q, kv in specs:
            Q = np.zeros(q * dim)
            K = np.zeros(kv * dim)
            V = np.zeros(kv * dim)
            lib.ref_make_toy_input(seed, q, kv, dim, ptr(Q), ptr(K), ptr(V))
            qs.append(Q), ks.append(K), vs.append(V), qr.append(q), kr.append(kv)
        Q, K, V = np.concatenate(qs), np.concatenate(ks), np.concatenate(vs)
        qr_a, kr_a = np.array(qr, dtype=np.int32), np.array(kr, dtype=np.int32)
        dec = np.zeros(Q.size)
        st = lib.ref_decomposed_attention(len(specs), dim, ptr(qr_a), ptr(kr_a), ptr(Q), ptr(K), ptr(V), width,
                                          ptr(dec))
        refo, qo, ko = [], 0, 0
        for q, kv in zip(qr, kr):
            o = np.zeros(q * dim)
            lib.ref_reference_attention(q, kv, dim, ptr(Q[qo * dim:]), ptr(K[ko * dim:]), ptr(V[ko * dim:]), ptr(o))
            refo.append(o)
            qo += q
            ko += kv
        return {"specs": [list(s) for s in specs], "width": width, "dim": dim, "status": st,
                "decomposed": dec.tolist(), "reference": np.concatenate(refo).tolist()}

    att.append(att_case([(21, 3, 6)], 1))
    att.append(att_case([(22, 3, 10), (23, 3, 2)], 2))
    att.append(att_case([(31, 2, 9), (32, 2, 4), (33, 2, 3)], 2))
    att.append(att_case([(61, 5, 37), (62, 5, 12), (63, 5, 80), (64, 5, 5)], 3, dim=64))
    for _ in range(100):
        n = int(rng.integers(1, 7))
        specs = [(int(rng.integers(0, 2**63)), int(rng.integers(1, 5)), int(rng.integers(1, 13))) for _ in range(n)]
        att.append(att_case(specs, int(rng.integers(1, n + 1))))
    g["attention"] = att
    # ---- acceptance
    acc = []
    for p in [0.0, 0.8, 1.0, 0.55]:
        out = np.zeros(64, dtype=np.int32)
        lib.ref_sample_accepted_prefix(p, 4, 77, 64, ptr(out))
        acc.append({"p": p, "window": 4, "seed": 77, "draws": out.tolist(),
                    "expected": lib.ref_expected_accepted_prefix(p, 4)})
    g["acceptance"] = acc
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump(g, f, separators=(",", ":"))
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


LBSS_OUT = os.path.join(os.path.dirname(OUT), "lbss_golden.json")
LBSS_CASES = [  # n, caps, alpha, beta, seed, slots
    (8, [8, 8], 8, 2, 2503, 40),
    (12, [4, 4, 4], 8, 2, 11, 40),
    (6, [2, 1, 2], 4, 2, 12, 30),
    (32, [32, 32, 32], 8, 2, 2503, 50),
    (20, [5, 20], 6, 3, 99, 45),
    (10, [3, 3, 3, 3], 4, 4, 7, 36),
]


def lbss_main():
    lib = load_ref()
    lib.ref_lbss_trace.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_ulonglong, C.c_int,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    rng = np.random.default_rng(31337)
    out = []
    for n, caps, alpha, beta, seed, slots in LBSS_CASES:
        m = len(caps)
        g = np.round(rng.uniform(1.0, 100.0, (n, m)), 3)
        if n == 32:
            g[:, 1] = g[:, 0]  # exact ties: lowest ssm id wins
        a = np.zeros((slots, n), np.int32)
        pw = np.zeros((slots, n), np.int32)
        ex = np.zeros(slots, np.int32)
        caps_a = np.array(caps, np.int32)
        gg = np.ascontiguousarray(g, dtype=np.float64)
        st = lib.ref_lbss_trace(n, m, ptr(caps_a), alpha, beta, seed, slots, ptr(gg), ptr(a), ptr(pw), ptr(ex))
        assert st == 0, st
        out.append({"n": n, "caps": caps, "alpha": alpha, "beta": beta, "seed": seed, "slots": slots,
                    "goodput": g.tolist(), "assignment": a.tolist(), "prewarm": pw.tolist(), "explore": ex.tolist()})
    with open(LBSS_OUT, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", LBSS_OUT, os.path.getsize(LBSS_OUT), "bytes")


TOY_OUT = os.path.join(os.path.dirname(OUT), "toy_bf16_golden.json")


def bf16_round(x):
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def toy_main():
    lib = load_ref()
    rng = np.random.default_rng(20240002)
    specs = [([(21, 3, 6)], 1, 4), ([(22, 3, 10), (23, 3, 2)], 2, 4), ([(31, 2, 9), (32, 2, 4), (33, 2, 3)], 2, 4),
             ([(61, 5, 37), (62, 5, 12), (63, 5, 80), (64, 5, 5)], 3, 64), ([(71, 8, 90), (72, 1, 33)], 1, 64),
             ([(81, 4, 40), (82, 4, 17), (83, 4, 29), (84, 2, 16), (85, 4, 1)], 2, 128)]
    for _ in range(30):
        n = int(rng.integers(1, 7))
        specs.append(([(int(rng.integers(0, 2**62)), int(rng.integers(1, 9)), int(rng.integers(1, 40)))
                       for _ in range(n)], int(rng.integers(1, n + 1)), int(rng.choice([4, 8, 64]))))
    out = []
    for spec, width, dim in specs:
        qs, ks, vs = [], [], []
        for seed, q, kv in spec:
            Q, K, V = np.zeros(q * dim), np.zeros(kv * dim), np.zeros(kv * dim)
            lib.ref_make_toy_input(seed, q, kv, dim, ptr(Q), ptr(K), ptr(V))
            qs.append(Q.astype(np.float32).astype(np.float64)), ks.append(bf16_round(K)), vs.append(bf16_round(V))
        Q, K, V = np.concatenate(qs), np.concatenate(ks), np.concatenate(vs)
        qr = np.array([s_[1] for s_ in spec], np.int32)
        kr = np.array([s_[2] for s_ in spec], np.int32)
        dec = np.zeros(Q.size)
        st = lib.ref_decomposed_attention(len(spec), dim, ptr(qr), ptr(kr), ptr(Q), ptr(K), ptr(V), width, ptr(dec))
        assert st == 0, st
        refo, qo, ko = [], 0, 0
        for q, kv in zip(qr, kr):
            o = np.zeros(q * dim)
            lib.ref_reference_attention(int(q), int(kv), dim, ptr(Q[qo * dim:]), ptr(K[ko * dim:]), ptr(V[ko * dim:]),
                                        ptr(o))
            refo.append(o)
            qo += q
            ko += kv
        out.append({"q_rows": qr.tolist(), "kv_rows": kr.tolist(), "width": width, "dim": dim, "q": Q.tolist(),
                    "k": K.tolist(), "v": V.tolist(), "decomposed": dec.tolist(),
                    "reference": np.concatenate(refo).tolist()})
    with open(TOY_OUT, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", TOY_OUT, os.path.getsize(TOY_OUT), "bytes")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "toy_bf16":
        toy_main()
    elif len(sys.argv) > 1 and sys.argv[1] == "lbss":
        lbss_main()
    else:
        main()
