"""Summarise SPIN_STAMPS timelines: per launch, CTA start spread, dependency-wait
release, main-loop end and last CTA end (us, relative to the first stamp)."""
import sys
from collections import defaultdict

import numpy as np

KIND = defaultdict(lambda: "?", {0: "qkv", 1: "attn", 2: "o", 3: "gate_up", 4: "down", 10: "T.qkv", 11: "T.o", 12: "T.gu", 13: "T.down", 14: "T.attn", 15: "lm_head", 16: "T.qkvepi", 17: "T.rn_o", 18: "T.swiglu", 19: "T.rn_dn"})
rows = defaultdict(list)
kinds = {}
with open(sys.argv[1]) as f:
    next(f)
    for line in f:
        l, k, c, *t = map(int, line.split(","))
        rows[l].append(t)
        kinds[l] = k
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
count = int(sys.argv[3]) if len(sys.argv) > 3 else 30
base = None
prev_end = None
agg = defaultdict(list)
for l in sorted(rows):
    t = np.array(rows[l], dtype=np.float64)
    t0 = t[:, 0][t[:, 0] > 0]
    t1 = t[:, 1][t[:, 1] > 0]
    t2 = t[:, 2][t[:, 2] > 0]
    t3 = t[:, 3][t[:, 3] > 0]
    if len(t0) == 0:
        continue
    if base is None:
        base = t0.min()
    s0, s1 = t0.min(), t0.max()
    w0 = t1.min() if len(t1) else np.nan
    w1 = t1.max() if len(t1) else np.nan
    m1 = t2.max() if len(t2) else np.nan
    e1 = t3.max() if len(t3) else np.nan
    gap = (w0 - prev_end) / 1e3 if prev_end is not None else np.nan
    agg[kinds[l]].append(((e1 - w0) / 1e3, gap, (w0 - s0) / 1e3, (m1 - w0) / 1e3))
    if first <= l < first + count:
        print(f"{l:4d} {KIND[kinds[l]]:8s} ctas={len(t0):4d} start {(s0-base)/1e3:8.2f}..{(s1-base)/1e3:8.2f} "
              f"wait_rel {(w0-base)/1e3:8.2f}..{(w1-base)/1e3:8.2f} main_end {(m1-base)/1e3:8.2f} "
              f"end {(e1-base)/1e3:8.2f}  gap_prev_end->wait {gap:6.2f}")
    prev_end = e1
print("kind: mean(end - wait_release), mean(prev end -> wait release), mean(start -> wait), mean(wait -> main end) [us]")
for k, v in sorted(agg.items()):
    a = np.nanmean(np.array(v), axis=0)
    print(f"  {KIND[k]:8s} n={len(v):4d} body={a[0]:6.2f} gap={a[1]:6.2f} prologue_lead={a[2]:6.2f} main={a[3]:6.2f}")
