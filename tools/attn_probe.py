"""Verify-attention probe: a 7B-shaped target with PROBE_LAYERS layers (default 2),
B = 32, gamma = 4, prompts U[128, 512]; one round, then the in-situ attention replay
(spin_kernel_bench kind 1). Prints us per launch; the target of ncu captures of the
verify attention kernel (attn_ws_kernel, or attn_kernel with SPIN_ATTN_WS=0)."""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2503_15921_b200.models import LLAMA_7B, LLAMA_68M, Engine, synthetic_prompts

tgt = dataclasses.replace(LLAMA_7B, n_layers=int(os.environ.get("PROBE_LAYERS", "2")))
B = 32
eng = Engine(tgt, (LLAMA_68M,), max_requests=B, max_ctx=640, window=4)
eng.prefill(range(B), synthetic_prompts(B, 128, 512, tgt.vocab, 2503))
slots = np.arange(B, dtype=np.int32)
eng.round(slots, np.zeros(B, np.int32))
us, by = eng.kernel_bench("attention", int(os.environ.get("PROBE_ITERS", "10")))
print(f"attention {us:.1f} us/launch {by / us / 1e3:.0f} GB/s ws={os.environ.get('SPIN_ATTN_WS', '1')}")
eng.close()
