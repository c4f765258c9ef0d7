import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2503_15921_b200.dist import shard
from paper_2503_15921_b200.models import LLAMA_7B, LLAMA_68M, LLAMA_160M, Engine, synthetic_prompts
N = 256
world, rank = int(os.environ.get("W", "2")), int(os.environ.get("R", "0"))
mine = shard(N, world, rank)
n_local = len(mine)
prompts = synthetic_prompts(N, 128, 512, LLAMA_7B.vocab, 2503 + 5)
eng = Engine(LLAMA_7B, (LLAMA_68M, LLAMA_160M), max_requests=n_local, max_ctx=704, window=4)
eng.prefill(range(n_local), [prompts[i] for i in mine])
slots = np.arange(n_local, dtype=np.int32)
print("prefilled", flush=True)
chosen, curve = eng.tune_micro_batches(slots, np.array([i % 2 for i in range(n_local)], np.int32), max_micro_batches=4, probe_rounds=3)
print("tuned", chosen, curve, flush=True)
