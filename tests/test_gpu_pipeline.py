"""Speculation/verification pipelining (the
reference's simulate_pipelined, pipeline.cpp:160-329, and tune_micro_batches,
:345-380). Outcome invariance (test_pipeline.cpp:234-249): micro-batched rounds
produce the oracle's serial-round tokens (tie-aware contract of tests/_parity.py),
and the overlapped device-resident loop produces exactly the tokens of the same
plan run slot by slot."""
import numpy as np
import pytest

from paper_2503_15921_b200.models import TINY_SSMS, TINY_TARGET, Engine, synthetic_prompts
from tests._parity import ParityRun

pytestmark = pytest.mark.gpu

B, W, CTX = 12, 4, 320


@pytest.mark.parametrize("mb", [[2, 2], [1, 3], [4, 1]])
def test_micro_batched_rounds_match_serial_oracle(mb):
    run = ParityRun(TINY_TARGET, TINY_SSMS, batch=B, prompt_lo=16, prompt_hi=64, seed=4242, window=W, max_ctx=CTX,
                    micro_batches=mb)
    plans = [np.array([0, 1] * 6, np.int32), np.array([1, 1, 0, -1, 0, 1, 0, 0, 1, 1, -1, 0], np.int32)]
    for r in range(8):
        g = run.round(plans[(r // 4) % 2])
        assert g["round_ms"] > 0 and g["verify_ms"] > 0
    run.check()
    run.close()


@pytest.mark.parametrize("mb", [[2, 2], [1, 2]])
def test_overlapped_loop_equals_slot_by_slot(mb):
    prompts = synthetic_prompts(B, 16, 64, TINY_TARGET.vocab, 77)
    dev = Engine(TINY_TARGET, TINY_SSMS, max_requests=B, max_ctx=CTX, window=W)
    host = Engine(TINY_TARGET, TINY_SSMS, max_requests=B, max_ctx=CTX, window=W)
    for e in (dev, host):
        e.prefill(range(B), prompts)
        e.set_micro_batches(mb)
    slots = np.arange(B, dtype=np.int32)
    assign = np.array([1, 0, 0, 1, 1, 0, 1, 0, 0, 0, 1, 1], np.int32)
    emitted, ms = dev.run_rounds(slots, assign, 8)
    per = [int(host.round(slots, assign)["accepted"].sum()) + B for _ in range(9)]
    assert list(emitted) == per[1:]  # run_rounds performs one host-driven round first
    assert ms > 0
    for s in range(B):
        assert np.array_equal(dev.tokens(s), host.tokens(s))
    dev.close()
    host.close()


def test_tune_micro_batches_measures_and_sets_plan():
    eng = Engine(TINY_TARGET, TINY_SSMS, max_requests=B, max_ctx=512, window=W)
    eng.prefill(range(B), synthetic_prompts(B, 16, 64, TINY_TARGET.vocab, 5))
    slots = np.arange(B, dtype=np.int32)
    assign = np.array([0, 1] * 6, np.int32)
    chosen, curve = eng.tune_micro_batches(slots, assign, max_micro_batches=3, probe_rounds=3)
    assert 1 <= len(curve) <= 3 and all(c > 0 for c in curve)
    assert np.array_equal(eng.micro_batches(), chosen)
    assert all(1 <= b <= 3 for b in chosen)
    eng.round(slots, assign)  # the chosen plan runs
    eng.close()
