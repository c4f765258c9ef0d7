"""Diagnostic: accumulation precision of the tcgen05 GEMM vs fp32 cuBLAS, both against fp64."""
import ctypes as C
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2503_15921_b200 import _lib

lib = _lib.load()
for n_out, k, t in [(768, 256, 40), (1376, 256, 40), (256, 688, 40), (4096, 4096, 160)]:
    g = torch.Generator().manual_seed(1)
    w = ((torch.rand((n_out, k), generator=g) * 2 - 1) * 0.1).to(torch.bfloat16)
    x = (torch.rand((t, k), generator=g) * 2 - 1).to(torch.bfloat16)
    ref = x.double() @ w.double().t()
    mp, grid, bn = C.c_int32(), C.c_int32(), C.c_int32()
    lib.spin_gemm_info(n_out, k, t, 0, C.byref(mp), C.byref(grid), C.byref(bn))
    part = torch.zeros((mp.value, t, n_out), dtype=torch.float32, device="cuda")
    wc, xc = w.cuda(), x.cuda()
    _lib.check(lib.spin_gemm(None, wc.data_ptr(), xc.data_ptr(), n_out, k, t, 0, part.data_ptr(), None, None, None))
    ours = part.sum(0).double().cpu()
    tfp32 = (xc.float() @ wc.float().t()).double().cpu()
    seq = (x.float().numpy().astype(np.float32)[:, None, :] * w.float().numpy()[None, :, :])
    rel = lambda a: ((a - ref).abs() / ref.abs().clamp_min(1e-3)).flatten()
    e1, e2 = rel(ours), rel(tfp32)
    print(f"{n_out}x{k}x{t}: ours med {e1.median():.2e} p99 {e1.quantile(0.99):.2e} max {e1.max():.2e} | "
          f"cublas-fp32 med {e2.median():.2e} p99 {e2.quantile(0.99):.2e} | abs ours {((ours-ref).abs()).max():.2e} cublas {((tfp32-ref).abs()).max():.2e}")
