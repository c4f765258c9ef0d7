"""Domain stickiness and per-domain acceptance of the config-4 domain models (13B target)."""
import os, sys
from dataclasses import replace
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2503_15921_b200.models import (LLAMA_13B_DOM, LLAMA_68M_DOM, LLAMA_160M_DOM, LLAMA_160M_B_DOM, Engine,
                                          domain_prompts)

B, W, R = 32, 4, 24
for gain in [float(g) for g in os.environ.get("GAINS", "12,20,28").split(",")]:
    tgt = replace(LLAMA_13B_DOM, planted_gain=gain)
    ssms = (LLAMA_68M_DOM, LLAMA_160M_DOM, LLAMA_160M_B_DOM)
    eng = Engine(tgt, ssms, max_requests=B, max_ctx=768, window=W)
    prompts = domain_prompts(B, 128, 512, tgt.vocab, 4, 2507)
    S = tgt.vocab // 4
    for j in range(3):
        eng.prefill(range(B), prompts)
        acc = np.zeros(B)
        for _ in range(R):
            acc += eng.round(np.arange(B, dtype=np.int32), np.full(B, j, np.int32))["accepted"]
        dom_stay = np.mean([np.mean(eng.tokens(i)[len(prompts[i]):] // S == i % 4) for i in range(B)])
        per_dom = [acc[[i for i in range(B) if i % 4 == d]].mean() / R for d in range(4)]
        print(f"gain {gain} ssm {j}: mean acc {acc.mean() / R:.2f} per domain {np.round(per_dom, 2)} "
              f"generated tokens in the prompt's domain {dom_stay:.2f}", flush=True)
    eng.close()
