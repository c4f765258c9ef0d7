"""GEMM timing probe: target GEMM replay (kernel_bench) on a 2-layer 7B-shaped target, B=32, gamma=4."""
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
import torch
torch.cuda.nvtx.range_push("bench")
tag = f"dbg={os.environ.get('SPIN_GEMM_DBG', '0')} fullk={int('SPIN_GEMM_FULLK' in os.environ)}"
for k in ("gemm",):
    us, by = eng.kernel_bench(k, 10)
    tag += f" | {k} {us:.1f}us {by / us / 1e3:.0f}GB/s"
torch.cuda.nvtx.range_pop()
print(tag)
eng.close()
