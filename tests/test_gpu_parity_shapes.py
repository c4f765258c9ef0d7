"""GPU-vs-oracle parity at the benchmarked model shapes:

* c2: LLaMA-7B-shaped target with the LLaMA-68M / 160M-shaped SSMs, 8 requests,
  3 rounds (hd=128 verify attention, K = 11008 down projection, vocab 32000);
* c3: the 7B shape with ragged draft lengths 1..16, packed AND padded, each
  against the oracle;
* c4: the LLaMA-13B shape with 3 heterogeneous SSMs, idle requests and an SSM
  switch.

Same contract as config 1 (tests/_parity.py): tokens bit-exact, logits within
1e-3 relative and 2x the measured fp32 reordering floor, near-tie adoptions
bounded by 2x that floor. Prompts are short (the CPU oracle runs a 7B / 13B
forward per round on the host cores); the GPU kernels are the production ones
at production shapes."""
import numpy as np
import pytest

from paper_2503_15921_b200.models import LLAMA_13B, LLAMA_160M, LLAMA_160M_B, LLAMA_68M, LLAMA_7B
from tests._parity import ParityRun, ragged_vs_oracle

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(1500)]


def test_c2_llama7b_shape_rounds_vs_oracle():
    run = ParityRun(LLAMA_7B, (LLAMA_68M, LLAMA_160M), batch=8, prompt_lo=16, prompt_hi=40, seed=7002, window=4,
                    max_ctx=96)
    assign = np.array([0, 1] * 4, np.int32)
    for _ in range(3):
        run.round(assign)
    st = run.check()
    run.close()
    print("c2-shape parity", st)


def test_c3_llama7b_shape_ragged_packed_and_padded_vs_oracle():
    out = ragged_vs_oracle(LLAMA_7B, (LLAMA_68M, LLAMA_160M), batch=16, window=16, width=0, prompt_lo=16,
                           prompt_hi=40, seed=7003, max_ctx=96)
    assert out["packed"]["query_rows"] == out["rows"] < out["padded"]["query_rows"]
    assert out["packed"]["kv_tokens"] < out["padded"]["kv_tokens"]
    print("c3-shape parity", out)


def test_c4_llama13b_shape_three_ssms_vs_oracle():
    run = ParityRun(LLAMA_13B, (LLAMA_68M, LLAMA_160M, LLAMA_160M_B), batch=4, prompt_lo=16, prompt_hi=32, seed=13002,
                    window=4, max_ctx=80)
    run.round([0, 1, 2, -1])
    run.round([2, 0, 1, 1])  # every request switches SSM (KV recompute on the destination)
    st = run.check()
    run.close()
    print("c4-shape parity", st)
