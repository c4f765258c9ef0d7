"""GEMM CTA timelines from SPIN_STAMPS (kinds 10-13 = target qkv/o/gate_up/down of layer 1,
8 stamps per CTA): start, producer wait release, first stage ready, last MMA issued,
first epilogue start, last epilogue done, end. Per launch: medians / max relative to the
earliest wait release (us)."""
import sys
from collections import defaultdict

import numpy as np

NAMES = {10: "qkv", 11: "o", 12: "gate_up", 13: "down"}
rows = defaultdict(list)
kinds = {}
with open(sys.argv[1]) as f:
    next(f)
    for line in f:
        l, k, c, *t = map(int, line.split(","))
        rows[l].append(t)
        kinds[l] = k
for l in sorted(rows):
    if kinds[l] not in NAMES:
        continue
    t = np.array(rows[l], dtype=np.float64).reshape(-1, 8)
    t = t[t[:, 0] > 0]
    base = t[:, 1].min()
    rel = (t - base) / 1e3
    print(f"{NAMES[kinds[l]]:8s} ctas={len(t)} start max {rel[:,0].max():6.2f} | wait rel med {np.median(rel[:,1]):6.2f} "
          f"| first stage med {np.median(rel[:,2]):6.2f} max {rel[:,2].max():6.2f} | last MMA med {np.median(rel[:,3]):6.2f} "
          f"max {rel[:,3].max():6.2f} | last epi done med {np.median(rel[:,5]):6.2f} max {rel[:,5].max():6.2f} "
          f"| end max {rel[:,6].max():6.2f}")

# per-CTA epilogue durations: first piece (start -> end), tail after the last MMA
for l in sorted(rows):
    if kinds[l] not in NAMES:
        continue
    t = np.array(rows[l], dtype=np.float64).reshape(-1, 8)
    t = t[t[:, 0] > 0]
    one = t[:, 7] >= t[:, 5] - 1  # single-piece CTAs: first epilogue is the last
    d1 = (t[:, 7] - t[:, 4]) / 1e3
    print(f"{NAMES[kinds[l]]:8s} first-piece epilogue med {np.median(d1[~one]) if (~one).any() else float('nan'):5.2f} "
          f"(multi-piece CTAs {int((~one).sum())}), single/last-piece epilogue med {np.median(d1[one]) if one.any() else float('nan'):5.2f}")
