"""Is a run_rounds divergence a near-tie or a bug? Compare host rounds and run_rounds vs the oracle."""
import sys
import numpy as np
sys.path.insert(0, '.')
from oracle import OracleEngine
from paper_2503_15921_b200.models import TINY_SSMS, TINY_TARGET, Engine, synthetic_prompts
B, W = 8, 4
prompts = synthetic_prompts(B, 16, 64, TINY_TARGET.vocab, 2503)
slots = np.arange(B, dtype=np.int32); assign = np.array([1, 0] * 4, np.int32)
cpu = OracleEngine(TINY_TARGET, TINY_SSMS, max_requests=B, max_ctx=256, window=W); cpu.prefill(range(B), prompts)
gh = Engine(TINY_TARGET, TINY_SSMS, max_requests=B, max_ctx=256, window=W, debug_logits=True); gh.prefill(range(B), prompts)
for r in range(7):
    c = cpu.round(slots, assign, want_logits=True); g = gh.round(slots, assign)
    lg = c["logits"]; top2 = np.sort(lg, 1)[:, -2:]; gap = top2[:, 1] - top2[:, 0]
    same = all(np.array_equal(g[k], c[k]) for k in ("drafts", "target", "accepted"))
    print(f"host round {r}: equal={same} min top-2 gap (oracle target logits) {gap.min():.2e}")
    if not same:
        for k in ("drafts", "target", "accepted"):
            if not np.array_equal(g[k], c[k]): print("  diff", k, np.argwhere(g[k] != c[k])[:4].tolist())
        break
