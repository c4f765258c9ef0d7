"""Deterministic prewarm stress: a fixed pseudo-random assignment per round, prewarm = the next
round's assignment, greedy rounds; prints a digest of every slot's committed tokens so runs with
different concurrency settings (environment) can be compared token for token."""
import hashlib, os, sys
from dataclasses import replace
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2503_15921_b200.models import (LLAMA_7B, LLAMA_13B_DOM, LLAMA_68M_DOM, LLAMA_160M_DOM, LLAMA_160M_B_DOM,
                                          Engine, domain_prompts)

B, W, R = 32, 4, int(os.environ.get("ROUNDS", "40"))
tgt = LLAMA_13B_DOM if os.environ.get("TGT") == "13b" else replace(LLAMA_7B, planted_domains=4, planted_gain=20.0)
ssms = (LLAMA_68M_DOM, LLAMA_160M_DOM, LLAMA_160M_B_DOM)
eng = Engine(tgt, ssms, max_requests=B, max_ctx=1024, window=W, use_graphs=os.environ.get("GRAPHS", "1") == "1", use_pdl=os.environ.get("PDL", "1") == "1")
eng.prefill(range(B), domain_prompts(B, 128, 512, tgt.vocab, 4, 7))
rng = np.random.default_rng(int(os.environ.get("SEED", "11")))
mode = os.environ.get("PLAN", "random")
if mode == "random":
    plans = [rng.integers(0, 3, B).astype(np.int32) for _ in range(R + 1)]
else:  # "split": drafting only on SSMs 0/1 in even rounds and SSM 2 in odd rounds, so a prewarm
    # never shares its SSM with a concurrent draft
    plans = [(rng.integers(0, 2, B) if r % 2 == 0 else np.full(B, 2)).astype(np.int32) for r in range(R + 1)]
slots = np.arange(B, dtype=np.int32)
err = None
verbose = os.environ.get("VERBOSE") == "1"
for r in range(R):
    pw = np.where(plans[r + 1] != plans[r], plans[r + 1], -1).astype(np.int32)
    if verbose:
        print(f"round {r} assign {plans[r].tolist()} prewarm {pw.tolist()}", file=sys.stderr, flush=True)
    try:
        eng.round(slots, plans[r], prewarm=pw)
    except Exception as e:
        err = f"round {r}: {e}"
        break
h = hashlib.sha256()
for i in range(B):
    h.update(eng.tokens(i).tobytes())
print("digest", h.hexdigest()[:16], "error", err)
