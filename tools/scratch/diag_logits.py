"""Diagnostic: where do GPU vs oracle target logits differ (config 1)?"""
import sys
import numpy as np
sys.path.insert(0, '.')
from oracle import OracleEngine
from paper_2503_15921_b200.models import TINY_SSMS, TINY_TARGET, Engine, synthetic_prompts

B, W = 8, 4
prompts = synthetic_prompts(B, 16, 64, TINY_TARGET.vocab, 2503)
gpu = Engine(TINY_TARGET, TINY_SSMS, max_requests=B, max_ctx=256, window=W, debug_logits=True)
cpu = OracleEngine(TINY_TARGET, TINY_SSMS, max_requests=B, max_ctx=256, window=W)
gpu.prefill(range(B), prompts)
cpu.prefill(range(B), prompts)
slots = np.arange(B, dtype=np.int32)
assign = np.array([0, 1] * 4, np.int32)
for r in range(6):
    g = gpu.round(slots, assign)
    c = cpu.round(slots, assign, want_logits=True)
    lg, lc = gpu.logits(B * (W + 1)), c["logits"]
    d = np.abs(lg - lc)
    rowmax = np.abs(lc).max(1)
    rel_row = d.max(1) / rowmax
    print(f"round {r}: max|c|={np.abs(lc).max():.3f} maxdiff={d.max():.4g} meddiff={np.median(d):.3g} "
          f"p99={np.quantile(d, 0.99):.3g} rel_row max={rel_row.max():.3g} med={np.median(rel_row):.3g}")
    print("   per-row maxdiff:", np.round(d.max(1), 5)[:15])
    print("   rel diff of top logit per row:", np.round(np.abs(lg.max(1) - lc.max(1)) / np.abs(lc.max(1)), 7)[:10])
