"""Config-3 packed verify timing for quick A/B runs (environment switches): one engine per pack
width in WIDTHS (default 16,32), 10 timed iterations after 3 warm-ups, microseconds per verify."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

from paper_2503_15921_b200.models import LLAMA_7B, LLAMA_68M, Engine, synthetic_prompts

B, W, SEED = 64, 16, 2503 + 3
rng = np.random.default_rng(SEED)
prompts = synthetic_prompts(B, 128, 512, LLAMA_7B.vocab, SEED)
lens = rng.integers(1, W + 1, B).astype(np.int32)
drafts = rng.integers(0, LLAMA_7B.vocab, int(lens.sum())).astype(np.int32)
out = []
for width in [int(x) for x in os.environ.get("WIDTHS", "16,32").split(",")]:
    eng = Engine(LLAMA_7B, (LLAMA_68M,), max_requests=B, max_ctx=576, window=W, pack_width=width)
    eng.prefill(range(B), prompts)
    slots = np.arange(B, dtype=np.int32)
    eng.verify_bench(slots, lens, drafts, packed=True, iters=3)
    r = eng.verify_bench(slots, lens, drafts, packed=True, iters=10)
    out.append((width, round(float(r["us"]))))
    eng.close()
print(os.environ.get("TAG", ""), out, flush=True)
