"""Prewarm must not change outcomes (bandit.cpp:122-139 prewarm_destination only moves the
switch cost): a fixed pseudo-random assignment per round over three domain SSMs of a
7B-shaped target, prewarm = the next round's SSM, run with and without prewarm -- committed
histories identical token for token. This configuration exposed catch-ups that reduced their
split-K pieces with a GEMM piece table still in flight on the legacy stream while the drafts
ran beside them (fixed by devattr.cpp upload_sync); it fails at round 10
without that fix."""
from dataclasses import replace

import numpy as np
import pytest

from paper_2503_15921_b200.models import (LLAMA_7B, LLAMA_68M_DOM, LLAMA_160M_B_DOM, LLAMA_160M_DOM, Engine,
                                          domain_prompts)

pytestmark = pytest.mark.gpu

B, W, R = 32, 4, 24


def _run(prewarm: bool, micro_batches=None):
    tgt = replace(LLAMA_7B, planted_domains=4, planted_gain=20.0)
    eng = Engine(tgt, (LLAMA_68M_DOM, LLAMA_160M_DOM, LLAMA_160M_B_DOM), max_requests=B, max_ctx=1024, window=W)
    if micro_batches is not None:
        eng.set_micro_batches(micro_batches)
    eng.prefill(range(B), domain_prompts(B, 128, 512, tgt.vocab, 4, 7))
    rng = np.random.default_rng(11)
    plans = [rng.integers(0, 3, B).astype(np.int32) for _ in range(R + 1)]
    slots = np.arange(B, dtype=np.int32)
    for r in range(R):
        pw = np.where(plans[r + 1] != plans[r], plans[r + 1], -1).astype(np.int32) if prewarm else None
        eng.round(slots, plans[r], prewarm=pw)
    toks = [eng.tokens(i).copy() for i in range(B)]
    eng.close()
    return toks


def test_prewarm_keeps_outcomes_under_concurrency():
    a, b = _run(True), _run(False)
    for i in range(B):
        assert np.array_equal(a[i], b[i]), i


def test_prewarm_keeps_outcomes_with_micro_batched_slots():
    """The same under f1 pipelining: micro-batched units per SSM (the catch-up waits for every
    SSM stream's last unit draft of the slot)."""
    a, b = _run(True, [2, 2, 2]), _run(False, [2, 2, 2])
    for i in range(B):
        assert np.array_equal(a[i], b[i]), i
