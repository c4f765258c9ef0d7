"""Does data written by one kernel stay in L2 for the next one under ncu --cache-control none?
A 28 MB fill followed by a read kernel (sum)."""
import torch
a = torch.empty(7 * 1024 * 1024, device="cuda")
for _ in range(3):
    a.fill_(1.0)
    s = a.sum()
torch.cuda.synchronize()
print(float(s))
