"""Packed ragged causal attention kernel (attention.cu) against a plain fp32
reference of the same op (numpy, on the same bf16 K/V). Device buffers through
libspin.so only."""
import numpy as np
import pytest

from paper_2503_15921_b200 import _lib
from tests._dev import DeviceBuffer, bf16_bits_to_f32, f32_to_bf16_bits

pytestmark = pytest.mark.gpu


def fp32_ref(q, kc, vc, layer, slots, qlens, kvlens, H, hd):
    out = np.zeros(q.shape, np.float32)
    r0 = 0
    for s, ql, kv in zip(slots, qlens, kvlens):
        for h in range(H):
            qq = q[r0:r0 + ql, h * hd:(h + 1) * hd]
            k = kc[layer, s, h, :kv]
            v = vc[layer, s, h, :kv]
            sc = (qq @ k.T) * np.float32(1.0 / np.sqrt(hd))
            pos = np.arange(kv)
            qpos = np.arange(kv - ql, kv)
            sc = np.where(pos[None, :] > qpos[:, None], -np.inf, sc)
            sc = np.exp(sc - sc.max(1, keepdims=True))
            out[r0:r0 + ql, h * hd:(h + 1) * hd] = (sc / sc.sum(1, keepdims=True)) @ v
        r0 += ql
    return out


def run(hd, H, L, S, ctx, layer, slots, qls, kvl, width, seed):
    rng = np.random.default_rng(seed)
    kb = f32_to_bf16_bits(rng.standard_normal((L, S, H, ctx, hd), dtype=np.float32))
    vb = f32_to_bf16_bits(rng.standard_normal((L, S, H, ctx, hd), dtype=np.float32))
    T = int(qls.sum())
    q = rng.standard_normal((T, H * hd), dtype=np.float32)
    kd, vd, qd = DeviceBuffer.from_array(kb), DeviceBuffer.from_array(vb), DeviceBuffer.from_array(q)
    od = DeviceBuffer(2 * T * H * hd)
    P = lambda a: a.ctypes.data_as(_lib.P_I32)
    _lib.check(_lib.load().spin_attention(None, H, hd, L, S, ctx, layer, kd.ptr, vd.ptr, qd.ptr, len(slots), P(slots),
                                          P(qls), P(kvl), width, od.ptr))
    out = bf16_bits_to_f32(od.download(np.uint16, (T, H * hd)))
    kc = bf16_bits_to_f32(kb).reshape(L, S, H, ctx, hd)
    vc = bf16_bits_to_f32(vb).reshape(L, S, H, ctx, hd)
    return out, fp32_ref(q, kc, vc, layer, slots, qls, kvl, H, hd)


@pytest.mark.parametrize("hd,H,width,qlen", [(128, 4, 0, 5), (64, 3, 0, 2), (128, 2, 3, 1), (64, 2, 5, 8),
                                             (128, 2, 0, 17)])
def test_attention_matches_fp32(hd, H, width, qlen):
    L, S, ctx = 2, 6, 700
    rng = np.random.default_rng(qlen)
    slots = np.array([4, 0, 2, 5, 1], np.int32)
    kvl = rng.integers(qlen, 650, len(slots)).astype(np.int32)
    kvl[1] = qlen  # a request that sees only its own queries
    qls = np.full(len(slots), qlen, np.int32)
    out, ref = run(hd, H, L, S, ctx, 1, slots, qls, kvl, width, hd + H + width + qlen)
    err = float(np.abs(out - ref).max())
    assert err <= 1e-2, err  # bf16 output rounding (|o| ~ 1)
    mism = float((out != bf16_bits_to_f32(f32_to_bf16_bits(ref))).mean())
    assert mism < 0.02, mism


@pytest.mark.parametrize("hd,qlen,width", [(128, 5, 3), (128, 8, 2), (64, 2, 3), (128, 12, 2)])
def test_attention_many_segments_per_row(hd, qlen, width):
    """Rows holding several segments whose tile counts are not multiples of the
    consumer-warp count (ring-stage ownership across segment boundaries)."""
    H, L, S, ctx = 2, 1, 12, 1100
    slots = np.arange(S, dtype=np.int32)[::-1].copy()
    kvl = np.array([37, 101, 1033, 64, 65, 200, 300, 33, 511, 97, 129, 700], np.int32)
    kvl = np.maximum(kvl, qlen).astype(np.int32)
    qls = np.full(S, qlen, np.int32)
    out, ref = run(hd, H, L, S, ctx, 0, slots, qls, kvl, width, 7 * hd + qlen)
    assert float(np.abs(out - ref).max()) <= 1e-2


@pytest.mark.parametrize("hd,width,qmax", [(128, 3, 17), (64, 2, 17), (128, 0, 17), (128, 4, 16), (64, 0, 12)])
def test_attention_ragged_windows(hd, width, qmax):
    """Mixed query counts in one launch (ragged drafts, config 3: attn_mq_kernel): warps whose
    8-query tile is empty for a piece pass its tiles on, split-KV pieces of 9..24-query requests
    meet at the named barrier and are merged by the last warp."""
    H, L, S, ctx = 3, 1, 10, 900
    rng = np.random.default_rng(hd + width + qmax)
    slots = rng.permutation(S).astype(np.int32)
    qls = np.minimum(np.array([1, 17, 9, 3, 16, 8, 12, 2, 17, 5], np.int32), qmax).astype(np.int32)
    kvl = np.maximum(rng.integers(20, 880, S), qls).astype(np.int32)
    kvl[3] = qls[3]  # a request that sees only its own queries
    out, ref = run(hd, H, L, S, ctx, 0, slots, qls, kvl, width, 11 * hd + width + qmax)
    assert float(np.abs(out - ref).max()) <= 1e-2
    mism = float((out != bf16_bits_to_f32(f32_to_bf16_bits(ref))).mean())
    assert mism < 0.02, mism
