import sys, dataclasses
import numpy as np
sys.path.insert(0, '.')
from oracle import OracleEngine
from paper_2503_15921_b200.models import TINY_SSMS, TINY_TARGET, Engine, synthetic_prompts
B, W = 8, 4
for name, tgt in [("resid0", dataclasses.replace(TINY_TARGET, resid_scale=0.0)), ("base", TINY_TARGET)]:
    prompts = synthetic_prompts(B, 16, 64, tgt.vocab, 2503)
    gpu = Engine(tgt, TINY_SSMS, max_requests=B, max_ctx=256, window=W, debug_logits=True)
    cpu = OracleEngine(tgt, TINY_SSMS, max_requests=B, max_ctx=256, window=W)
    gpu.prefill(range(B), prompts); cpu.prefill(range(B), prompts)
    g = gpu.round(np.arange(B, dtype=np.int32), np.array([0, 1] * 4, np.int32))
    c = cpu.round(np.arange(B, dtype=np.int32), np.array([0, 1] * 4, np.int32), want_logits=True)
    d = np.abs(gpu.logits(B * (W + 1)) - c["logits"])
    print(name, "maxdiff", d.max(), "median", np.median(d))
