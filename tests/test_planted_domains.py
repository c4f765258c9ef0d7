"""Token domains of the synthetic planted map (spin_c.h planted_domains / planted_mask):
the oracle's map keeps every domain, is a permutation inside it, reduces to the one-domain
map pi(t) = (A t + C) mod V, and an SSM's lm_head carries the planted term only on its
domains. CPU only (the oracle); the GPU engine is pinned to the same weights by the
parity test in tests/test_gpu_engine_parity.py."""
import ctypes as C
from dataclasses import replace

import numpy as np

import oracle
from paper_2503_15921_b200.models import LLAMA_68M_DOM, LLAMA_13B_DOM, TINY_TARGET, domain_prompts


def _next(shape, toks):
    lib = oracle.load_oracle()
    d = oracle.so_desc(shape)
    return np.array([lib.so_planted_next(C.byref(d), int(t)) for t in toks])


def test_one_domain_is_the_round1_map():
    V = TINY_TARGET.vocab
    a = 7919 % V
    while np.gcd(a, V) != 1:
        a += 1
    t = np.arange(V)
    assert (_next(TINY_TARGET, t) == (a * t + 12345 % V) % V).all()
    assert (_next(replace(TINY_TARGET, planted_domains=1), t) == _next(TINY_TARGET, t)).all()


def test_domain_map_is_a_permutation_of_each_domain():
    shape = replace(TINY_TARGET, planted_domains=4)
    V, S = shape.vocab, shape.vocab // 4
    nxt = _next(shape, np.arange(V))
    for d in range(4):
        block = nxt[d * S:(d + 1) * S]
        assert ((block >= d * S) & (block < (d + 1) * S)).all()
        assert len(np.unique(block)) == S


def test_mask_selects_planted_lm_head_rows():
    lib = oracle.load_oracle()
    lib.so_weight_bits.restype = C.c_uint16
    lib.so_weight_bits.argtypes = [C.POINTER(oracle.SoModelDesc), C.c_int, C.c_int, C.c_int64, C.c_int64]
    base = replace(TINY_TARGET, planted_domains=4)
    only1 = replace(base, planted_mask=0b0010)
    unplanted = replace(base, planted_gain=0.0)
    S = base.vocab // 4
    for row in (3, S + 5, 2 * S + 7, 3 * S + 11):
        dom = row // S
        bits = [lib.so_weight_bits(C.byref(oracle.so_desc(m)), 2, 0, row, 17) for m in (base, only1, unplanted)]
        assert bits[0] != bits[2]  # every domain planted in the target
        assert (bits[1] == bits[0]) if dom == 1 else (bits[1] == bits[2])


def test_domain_prompts_stay_in_their_domain():
    ps = domain_prompts(8, 16, 40, LLAMA_13B_DOM.vocab, 4, 7)
    S = LLAMA_13B_DOM.vocab // 4
    for i, p in enumerate(ps):
        assert ((p // S) == i % 4).all()
    assert LLAMA_68M_DOM.planted_domains == LLAMA_13B_DOM.planted_domains
