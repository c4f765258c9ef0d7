"""Profiling driver: config-2 engine, prefill, warm rounds, then one round
inside an NVTX range "round" (for ncu --nvtx-include round/).
  --graph 0  issue the profiled round kernel by kernel (no CUDA graph)"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2503_15921_b200.models import LLAMA_7B, LLAMA_68M, LLAMA_160M, Engine, synthetic_prompts

ap = argparse.ArgumentParser()
ap.add_argument("--graph", type=int, default=1)
ap.add_argument("--warm", type=int, default=2)
ap.add_argument("--pack-width", type=int, default=0)
a = ap.parse_args()
B, W = 32, 4
eng = Engine(LLAMA_7B, (LLAMA_68M, LLAMA_160M), max_requests=B, max_ctx=640, window=W, use_graphs=bool(a.graph),
             pack_width=a.pack_width)
eng.prefill(range(B), synthetic_prompts(B, 128, 512, LLAMA_7B.vocab, 2503))
slots = np.arange(B, dtype=np.int32)
assign = np.array([i % 2 for i in range(B)], np.int32)
for _ in range(a.warm):
    eng.round(slots, assign)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("round")
out = eng.round(slots, assign)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("round_ms", out["round_ms"], "verify_ms", out["verify_ms"], "draft_ms", out["draft_ms"])
