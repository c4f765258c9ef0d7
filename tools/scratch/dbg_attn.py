import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2503_15921_b200 import _lib
from tests.test_gpu_attention import torch_ref
lib = _lib.load()
P = lambda a: a.ctypes.data_as(_lib.P_I32)
for hd, H, qlen, kvs in [(128, 1, 1, [32]), (128, 1, 1, [40]), (128, 1, 2, [64]), (128, 1, 5, [200]), (64, 1, 2, [64])]:
    g = torch.Generator().manual_seed(0)
    L, S, ctx = 1, 2, 256
    kc = torch.randn((L, S, H, ctx, hd), generator=g).to(torch.bfloat16).cuda()
    vc = torch.randn((L, S, H, ctx, hd), generator=g).to(torch.bfloat16).cuda()
    slots = np.array([1], np.int32); kvl = np.array(kvs, np.int32); qls = np.array([qlen], np.int32)
    q = torch.randn((qlen, H * hd), generator=g).cuda()
    out = torch.empty((qlen, H * hd), dtype=torch.bfloat16, device="cuda")
    _lib.check(lib.spin_attention(None, H, hd, L, S, ctx, 0, kc.data_ptr(), vc.data_ptr(), q.data_ptr(), 1, P(slots), P(qls), P(kvl), 0, out.data_ptr()))
    torch.cuda.synchronize()
    ref = torch_ref(q, kc, vc, 0, slots, qls, kvl, H, hd)
    d = (out.float() - ref).abs()
    print(hd, qlen, kvs, "maxerr", d.max().item(), "bad dims", (d > 1e-2).nonzero()[:8].tolist())
    print("  out", out.float()[0, :6].tolist()); print("  ref", ref[0, :6].tolist())
