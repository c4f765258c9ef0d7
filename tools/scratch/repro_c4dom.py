"""Repro: LBSS serve loop with domain-planted SSMs (c4 setup) on a small target."""
import os, sys
from dataclasses import replace
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2503_15921_b200.models import (TINY_TARGET, LLAMA_68M_DOM, LLAMA_160M_DOM, LLAMA_160M_B_DOM, Engine,
                                          domain_prompts)
from paper_2503_15921_b200.selector import Lbss
import bench

B, W = 32, 4
from paper_2503_15921_b200.models import LLAMA_13B_DOM, LLAMA_7B
tgt = {"13b": LLAMA_13B_DOM, "7b": replace(LLAMA_7B, planted_domains=4)}.get(os.environ.get("TGT", ""), replace(TINY_TARGET, vocab=32000, planted_domains=4))
ssms = (LLAMA_68M_DOM, LLAMA_160M_DOM, LLAMA_160M_B_DOM)
slots_n = int(os.environ.get("SLOTS", "64"))
max_ctx = ((512 + (W + 1) * (slots_n + 4) + 8 + 63) // 64) * 64
prompts = domain_prompts(B, 128, 512, tgt.vocab, 4, 7)
eng = Engine(tgt, ssms, max_requests=B, max_ctx=max_ctx, window=W, use_graphs=os.environ.get("GRAPHS", "1") == "1", use_pdl=os.environ.get("PDL", "1") == "1")
eng.prefill(range(B), prompts)
sel = Lbss(B, [B] * 3, alpha=8, beta=2, seed=1)
rep, final = bench.serve(eng, sel, B, 3, np.arange(B, dtype=np.int32), slots_n, prewarm=os.environ.get("PREWARM", "1") == "1")
print(rep, np.bincount(final[final >= 0], minlength=3))
