"""GPU-vs-oracle logit distance next to the oracle's own accumulation-order noise floor (config 1)."""
import sys
import numpy as np
sys.path.insert(0, '.')
import oracle
from oracle import OracleEngine
from paper_2503_15921_b200.models import TINY_SSMS, TINY_TARGET, Engine, synthetic_prompts
B, W, R = 8, 4, 16
lib = oracle.load_oracle()
prompts = synthetic_prompts(B, 16, 64, TINY_TARGET.vocab, 2503)
slots, assign = np.arange(B, dtype=np.int32), np.array([0, 1] * 4, np.int32)
runs = {}
for name in ("gpu", "cpu16", "cpu8"):
    if name == "gpu":
        e = Engine(TINY_TARGET, TINY_SSMS, max_requests=B, max_ctx=256, window=W, debug_logits=True)
    else:
        lib.so_set_gemm_lanes(16 if name == "cpu16" else 8)
        e = OracleEngine(TINY_TARGET, TINY_SSMS, max_requests=B, max_ctx=256, window=W)
    e.prefill(range(B), prompts)
    lg = []
    for r in range(R):
        o = e.round(slots, assign) if name == "gpu" else e.round(slots, assign, want_logits=True)
        lg.append(e.logits(B * (W + 1)) if name == "gpu" else o["logits"])
    runs[name] = lg
def dist(a, b):
    return max(np.abs(x - y).max() / np.abs(y).max() for x, y in zip(a, b))
print("gpu vs cpu16", dist(runs["gpu"], runs["cpu16"]), "cpu8 vs cpu16", dist(runs["cpu8"], runs["cpu16"]))
