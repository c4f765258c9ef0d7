import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2503_15921_b200.models import *
big = os.environ.get("BIG") == "1"
tgt, ssms = (LLAMA_7B, (LLAMA_68M, LLAMA_160M)) if big else (TINY_TARGET, TINY_SSMS)
n = int(os.environ.get("N", "128"))
eng = Engine(tgt, ssms, max_requests=n, max_ctx=768 if big else 512, window=4)
eng.prefill(range(n), synthetic_prompts(n, int(os.environ.get('PLO', 128 if big else 16)), int(os.environ.get('PHI', 512 if big else 64)), tgt.vocab, 5))
slots = np.arange(n, dtype=np.int32)
assign = np.array([i % 2 for i in range(n)], np.int32)
for mb in ([2, 2], [1, 2], [3, 3], [4, 4]):
    eng.set_micro_batches(mb)
    r = eng.round(slots, assign)
    e, ms = eng.run_rounds(slots, assign, 3)
    print(mb, "ok", e, ms, flush=True)
eng.close()
