"""tcgen05 GEMM (gemm.cu) against a plain PyTorch fp32 reference of the same op."""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2503_15921_b200 import _lib


def _info(n_out, k, t, mode):
    mp, grid, bn = C.c_int32(), C.c_int32(), C.c_int32()
    _lib.check(_lib.load().spin_gemm_info(n_out, k, t, mode, C.byref(mp), C.byref(grid), C.byref(bn)))
    return mp.value, grid.value, bn.value


def _rand(shape, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return (torch.rand(shape, generator=g) * 2 - 1).to(torch.bfloat16).cuda()


@pytest.mark.parametrize(
    "n_out,k,t",
    [(256, 256, 16), (1376, 256, 40), (768, 688, 8), (4096, 4096, 160), (12288, 4096, 160), (4096, 11008, 160),
     (22016, 4096, 160), (2304, 768, 32), (1024, 512, 600)],
)
def test_gemm_partial_matches_torch(n_out, k, t):
    lib = _lib.load()
    w = _rand((n_out, k), 1) * 0.05
    x = _rand((t, k), 2)
    mp, grid, bn = _info(n_out, k, t, 0)
    part = torch.zeros((mp, t, n_out), dtype=torch.float32, device="cuda")
    _lib.check(lib.spin_gemm(None, w.data_ptr(), x.data_ptr(), n_out, k, t, 0, part.data_ptr(), None, None, None))
    torch.cuda.synchronize()
    got = part.sum(0)
    ref = x.float() @ w.float().t()
    err = (got - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= 1e-4 * scale + 1e-5, f"max err {err} (scale {scale}, pieces {mp}, grid {grid}, bn {bn})"


@pytest.mark.parametrize("n_out,k,t", [(4096, 256, 40), (32000, 4096, 160), (1000, 128, 5), (2048, 256, 520)])
def test_gemm_argmax_matches_torch(n_out, k, t):
    lib = _lib.load()
    w = _rand((n_out, k), 3)
    x = _rand((t, k), 4)
    n_mt = (n_out + 127) // 128
    val = torch.empty((n_mt, t), dtype=torch.float32, device="cuda")
    idx = torch.empty((n_mt, t), dtype=torch.int32, device="cuda")
    logits = torch.empty((t, n_out), dtype=torch.float32, device="cuda")
    _lib.check(lib.spin_gemm(None, w.data_ptr(), x.data_ptr(), n_out, k, t, 1, None, val.data_ptr(), idx.data_ptr(),
                             logits.data_ptr()))
    torch.cuda.synchronize()
    ref = x.float() @ w.float().t()
    assert (logits - ref).abs().max().item() <= 1e-4 * ref.abs().max().item()
    # per-tile argmax of the kernel's own logits, lowest index on ties
    best = val.max(0)
    tile = best.indices
    got_idx = idx.gather(0, tile[None, :].long())[0]
    exp_idx = logits.argmax(1).int()
    assert torch.equal(got_idx, exp_idx)
    assert torch.equal(best.values, logits.max(1).values)
