"""Config-3 packed verify (7B target, 64 requests, ragged windows U{1..16}, pack width 16) for a
kernel launch list: ncu --metrics gpu__time_duration.sum --csv python tools/c3_profile.py;
tools/launch_summary.py summarises the CSV."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2503_15921_b200.models import LLAMA_7B, LLAMA_68M, Engine, synthetic_prompts

B, W, SEED = 64, 16, 2503 + 3
rng = np.random.default_rng(SEED)
prompts = synthetic_prompts(B, 128, 512, LLAMA_7B.vocab, SEED)
lens = rng.integers(1, W + 1, B).astype(np.int32)
drafts = rng.integers(0, LLAMA_7B.vocab, int(lens.sum())).astype(np.int32)
eng = Engine(LLAMA_7B, (LLAMA_68M,), max_requests=B, max_ctx=576, window=W, pack_width=16)
eng.prefill(range(B), prompts)
eng.verify_bench(np.arange(B, dtype=np.int32), lens, drafts, packed=True, iters=int(os.environ.get("ITERS", "1")))
