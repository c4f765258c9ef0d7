"""Packed ragged causal attention kernel (attention.cu) against a plain PyTorch
fp32 reference of the same op."""
import numpy as np
import pytest

from paper_2503_15921_b200 import _lib

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def torch_ref(q, kc, vc, layer, slots, qlens, kvlens, H, hd):
    out = torch.zeros(q.shape, dtype=torch.float32, device=q.device)
    r0 = 0
    for s, ql, kv in zip(slots, qlens, kvlens):
        for h in range(H):
            qq = q[r0:r0 + ql, h * hd:(h + 1) * hd].float()
            k = kc[layer, s, h, :kv].float()
            v = vc[layer, s, h, :kv].float()
            sc = (qq @ k.t()) * (1.0 / np.sqrt(hd))
            pos = torch.arange(kv, device=q.device)
            qpos = torch.arange(kv - ql, kv, device=q.device)
            sc = sc.masked_fill(pos[None, :] > qpos[:, None], float("-inf"))
            out[r0:r0 + ql, h * hd:(h + 1) * hd] = torch.softmax(sc, -1) @ v
        r0 += ql
    return out


@pytest.mark.parametrize("hd,H,width,qlen", [(128, 4, 0, 5), (64, 3, 0, 2), (128, 2, 3, 1), (64, 2, 5, 8),
                                             (128, 2, 0, 17)])
def test_attention_matches_torch(hd, H, width, qlen):
    g = torch.Generator(device="cpu").manual_seed(hd + H + width + qlen)
    L, S, ctx = 2, 6, 700
    kc = torch.randn((L, S, H, ctx, hd), generator=g).to(torch.bfloat16).cuda()
    vc = torch.randn((L, S, H, ctx, hd), generator=g).to(torch.bfloat16).cuda()
    rng = np.random.default_rng(qlen)
    slots = np.array([4, 0, 2, 5, 1], np.int32)
    kvl = rng.integers(qlen, 650, len(slots)).astype(np.int32)
    kvl[1] = qlen  # a request that sees only its own queries
    qls = np.full(len(slots), qlen, np.int32)
    T = int(qls.sum())
    q = torch.randn((T, H * hd), generator=g).cuda()
    out = torch.empty((T, H * hd), dtype=torch.bfloat16, device="cuda")
    lib = _lib.load()
    P = lambda a: a.ctypes.data_as(_lib.P_I32)
    _lib.check(lib.spin_attention(None, H, hd, L, S, ctx, 1, kc.data_ptr(), vc.data_ptr(), q.data_ptr(), len(slots),
                                  P(slots), P(qls), P(kvl), width, out.data_ptr()))
    ref = torch_ref(q, kc, vc, 1, slots, qls, kvl, H, hd)
    err = (out.float() - ref).abs().max().item()
    assert err <= 1e-2, err  # bf16 output rounding (|o| ~ 1)
    mism = (out.float() != ref.to(torch.bfloat16).float()).float().mean().item()
    assert mism < 0.02, mism


@pytest.mark.parametrize("hd,qlen,width", [(128, 5, 3), (128, 8, 2), (64, 2, 3), (128, 12, 2)])
def test_attention_many_segments_per_row(hd, qlen, width):
    """Rows holding several segments whose tile counts are not multiples of the
    consumer-warp count (ring-stage ownership across segment boundaries)."""
    g = torch.Generator(device="cpu").manual_seed(7 * hd + qlen)
    H, L, S, ctx = 2, 1, 12, 1100
    kc = torch.randn((L, S, H, ctx, hd), generator=g).to(torch.bfloat16).cuda()
    vc = torch.randn((L, S, H, ctx, hd), generator=g).to(torch.bfloat16).cuda()
    slots = np.arange(S, dtype=np.int32)[::-1].copy()
    kvl = np.array([37, 101, 1033, 64, 65, 200, 300, 33, 511, 97, 129, 700], np.int32)
    kvl = np.maximum(kvl, qlen).astype(np.int32)
    qls = np.full(S, qlen, np.int32)
    q = torch.randn((int(qls.sum()), H * hd), generator=g).cuda()
    out = torch.empty((int(qls.sum()), H * hd), dtype=torch.bfloat16, device="cuda")
    P = lambda a: a.ctypes.data_as(_lib.P_I32)
    _lib.check(_lib.load().spin_attention(None, H, hd, L, S, ctx, 0, kc.data_ptr(), vc.data_ptr(), q.data_ptr(), S,
                                          P(slots), P(qls), P(kvl), width, out.data_ptr()))
    ref = torch_ref(q, kc, vc, 0, slots, qls, kvl, H, hd)
    assert (out.float() - ref).abs().max().item() <= 1e-2
