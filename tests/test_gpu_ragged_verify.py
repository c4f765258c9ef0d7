"""Config 3: ragged draft lengths, packed (request decomposition) vs padded
verification. Each of the two must produce the oracle's target tokens on every
real query row (tie-aware against the measured fp32 floor, tests/_parity.py),
and the packed step must process fewer rows / KV tokens (slot_engine.cpp:24-45
verify_batch_cost)."""
import numpy as np
import pytest

from paper_2503_15921_b200.models import TINY_SSMS, TINY_TARGET, Engine, synthetic_prompts
from tests._parity import ragged_vs_oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("B,W,width", [(8, 16, 0), (12, 8, 3), (5, 4, 0)])
def test_packed_equals_padded_tokens(B, W, width):
    rng = np.random.default_rng(B + W)
    eng = Engine(TINY_TARGET, TINY_SSMS, max_requests=B, max_ctx=256, window=W, pack_width=width,
                 debug_logits=False)
    eng.prefill(range(B), synthetic_prompts(B, 16, 64, TINY_TARGET.vocab, 31 + B))
    slots = np.arange(B, dtype=np.int32)
    lens = rng.integers(1, W + 1, B).astype(np.int32)
    drafts = rng.integers(0, TINY_TARGET.vocab, int(lens.sum())).astype(np.int32)
    p = eng.verify_bench(slots, lens, drafts, packed=True, iters=2)
    q = eng.verify_bench(slots, lens, drafts, packed=False, iters=2)
    eng.close()
    assert p["real_rows"] == q["real_rows"] == int((lens + 1).sum())
    assert p["query_rows"] == p["real_rows"]
    assert q["query_rows"] == B * (int(lens.max()) + 1)
    assert p["kv_tokens"] <= q["kv_tokens"]


@pytest.mark.parametrize("B,W,width", [(8, 16, 0), (12, 8, 3), (5, 4, 0), (24, 16, 6)])
def test_packed_and_padded_match_oracle(B, W, width):
    out = ragged_vs_oracle(TINY_TARGET, TINY_SSMS, batch=B, window=W, width=width, prompt_lo=16, prompt_hi=64,
                           seed=31 + B, max_ctx=256)
    assert out["packed"]["query_rows"] == out["rows"]
    print("c1-shape ragged parity", out)


def test_ragged_verify_rejects_bad_lengths():
    from paper_2503_15921_b200._lib import SpinError

    eng = Engine(TINY_TARGET, TINY_SSMS, max_requests=4, max_ctx=128, window=4)
    eng.prefill(range(4), synthetic_prompts(4, 16, 32, TINY_TARGET.vocab, 5))
    with pytest.raises(SpinError):
        eng.verify_bench(np.arange(4, dtype=np.int32), np.array([1, 5, 2, 2], np.int32))
    eng.close()
