"""Draft-phase time of the config-2 round with both SSMs drafting (i % 2) vs the 160M SSM alone
on its 16 requests (the 68M's requests idle): how much the concurrent 68M drafts cost the
critical 160M chain. Prints median draft / verify ms over ROUNDS rounds per assignment."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

from paper_2503_15921_b200.models import LLAMA_7B, LLAMA_68M, LLAMA_160M, Engine, synthetic_prompts

B, W, R = 32, 4, int(os.environ.get("ROUNDS", "12"))
eng = Engine(LLAMA_7B, (LLAMA_68M, LLAMA_160M), max_requests=B, max_ctx=1024, window=W)
eng.prefill(range(B), synthetic_prompts(B, 128, 512, LLAMA_7B.vocab, 2503))
slots = np.arange(B, dtype=np.int32)
for name, ssm_of in (("both", np.array([i % 2 for i in range(B)], np.int32)),
                     ("160M alone", np.array([1 if i % 2 else -1 for i in range(B)], np.int32)),
                     ("68M alone", np.array([0 if i % 2 == 0 else -1 for i in range(B)], np.int32)),
                     ("both", np.array([i % 2 for i in range(B)], np.int32))):
    d, v = [], []
    for r in range(R):
        o = eng.round(slots, ssm_of)
        if r >= 2:
            d.append(o["draft_ms"]), v.append(o["verify_ms"])
    print(f"{name:12s} draft {np.median(d):.3f} ms verify {np.median(v):.3f} ms", flush=True)
