import numpy as np, sys
from collections import defaultdict
rows=defaultdict(list); kinds={}
with open(sys.argv[1]) as f:
    next(f)
    for line in f:
        l,k,c,*t=map(int,line.split(',')); rows[l].append(t); kinds[l]=k
def span(l):
    t=np.array(rows[l],dtype=float); t0=t[:,0][t[:,0]>0]; t3=t[:,3][t[:,3]>0]
    return t0.min(), t3.max() if len(t3) else np.nan
for step in range(4):
    first=40+step*60; last=first+59
    s0,_=span(first); _,e1=span(last)
    print(f"step {step}: layers {(e1-s0)/1e3:.1f} us")
