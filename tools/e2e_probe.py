"""Host overhead of the public per-slot round call: wall time of eng.round() vs the
device round time it reports (config 2)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2503_15921_b200.models import LLAMA_7B, LLAMA_68M, LLAMA_160M, Engine, synthetic_prompts

B, W = 32, 4
eng = Engine(LLAMA_7B, (LLAMA_68M, LLAMA_160M), max_requests=B, max_ctx=1024, window=W)
eng.prefill(range(B), synthetic_prompts(B, 128, 512, LLAMA_7B.vocab, 2503))
slots = np.arange(B, dtype=np.int32)
assign = np.array([i % 2 for i in range(B)], np.int32)
for _ in range(3):
    eng.round(slots, assign)
walls, devs = [], []
for _ in range(20):
    t0 = time.perf_counter()
    out = eng.round(slots, assign)
    walls.append((time.perf_counter() - t0) * 1e3)
    devs.append(out["round_ms"])
w, d = np.median(walls), np.median(devs)
print(f"round() wall {w:.3f} ms, device {d:.3f} ms, host overhead {w - d:.3f} ms")
emitted, ms = eng.run_rounds(slots, assign, 10)
print(f"run_rounds: {ms / 10:.3f} ms per round")
