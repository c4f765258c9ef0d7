"""Attention CTA timelines from SPIN_STAMPS (kind 1, 8 stamps per CTA, warp 0):
start, wait release, first tile ready, q ready, piece-0 tile loop end, piece-0 partial
stored, merge start, end. Medians over launches of per-launch max / median (us,
relative to the launch's first wait release) and of the last CTA's phases."""
import sys
from collections import defaultdict

import numpy as np

rows = defaultdict(list)
kinds = {}
with open(sys.argv[1]) as f:
    next(f)
    for line in f:
        l, k, c, *t = map(int, line.split(","))
        rows[l].append(t)
        kinds[l] = k
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
KIND = int(sys.argv[3]) if len(sys.argv) > 3 else 1
res = defaultdict(list)
for l in sorted(rows):
    if kinds[l] != KIND or l < first:
        continue
    t = np.array(rows[l], dtype=float).reshape(-1, 8)
    t = t[t[:, 0] > 0]
    w = t[:, 1][t[:, 1] > 0]
    if not len(w):
        continue
    base = w.min()
    res["ctas"].append(len(t))
    res["wait spread"].append((w.max() - base) / 1e3)
    for i, n in [(4, "loop end"), (5, "stored"), (6, "merge start"), (7, "end")]:
        v = t[:, i][t[:, i] > 0]
        res[n + " max"].append((v.max() - base) / 1e3 if len(v) else np.nan)
        res[n + " med"].append((np.median(v) - base) / 1e3 if len(v) else np.nan)
    r = t[np.argmax(t[:, 7])]
    res["last CTA: wait->loop end"].append((r[4] - r[1]) / 1e3 if r[1] > 0 and r[4] > 0 else np.nan)
    res["last CTA: loop end->stored"].append((r[5] - r[4]) / 1e3 if r[5] > 0 and r[4] > 0 else np.nan)
    res["last CTA: stored->end"].append((r[7] - r[5]) / 1e3 if r[5] > 0 else np.nan)
    res["last CTA: merge"].append((r[7] - r[6]) / 1e3 if r[6] > 0 else np.nan)
for n, v in res.items():
    print(f"{n:28s} {np.nanmedian(v):7.2f}")
