"""Target layer-1 timeline from SPIN_STAMPS (kinds 10-19): per launch, first CTA start,
dependency release (first), last stamp; the gap from the previous launch's last stamp to
this launch's first release, and the body (release -> last stamp) [us]."""
import sys
from collections import defaultdict

import numpy as np

NAMES = {10: "qkv", 16: "qkv_epi", 14: "attn", 11: "o", 17: "resid_norm(o)", 12: "gate_up", 18: "swiglu",
         13: "down", 19: "resid_norm(down)"}
rows = defaultdict(list)
kinds = {}
with open(sys.argv[1]) as f:
    next(f)
    for line in f:
        l, k, c, *t = map(int, line.split(","))
        rows[l].append(t)
        kinds[l] = k
prev = None
tot = defaultdict(float)
for l in sorted(rows):
    if kinds[l] not in NAMES:
        continue
    t = np.array(rows[l], dtype=np.float64)
    per = 8 if kinds[l] in (10, 11, 12, 13, 14) else 4
    t = t.reshape(-1, per)
    t = t[t[:, 0] > 0]
    start, rel = t[:, 0].min(), t[:, 1][t[:, 1] > 0].min()
    end = t[t > 0].max()
    gap = (rel - prev) / 1e3 if prev is not None else float("nan")
    body = (end - rel) / 1e3
    print(f"{NAMES[kinds[l]]:17s} blocks={len(t):5d} start->release {(rel-start)/1e3:6.2f}  gap {gap:6.2f}  body {body:6.2f}")
    if prev is not None:
        tot["gaps"] += gap
    tot[NAMES[kinds[l]]] += body
    prev = end
print("sum:", {k: round(v, 2) for k, v in tot.items()}, "layer", round(sum(tot.values()), 2))
