"""tcgen05 GEMM (gemm.cu) against a plain fp32 reference of the same op (numpy,
on the same bf16-rounded operands). Device buffers through libspin.so only."""
import ctypes as C

import numpy as np
import pytest

from paper_2503_15921_b200 import _lib
from tests._dev import DeviceBuffer, bf16_bits_to_f32, f32_to_bf16_bits

pytestmark = pytest.mark.gpu


def _info(n_out, k, t, mode):
    mp, grid, bn = C.c_int32(), C.c_int32(), C.c_int32()
    _lib.check(_lib.load().spin_gemm_info(n_out, k, t, mode, C.byref(mp), C.byref(grid), C.byref(bn)))
    return mp.value, grid.value, bn.value


def _rand_bf16(shape, seed, scale=1.0):
    r = np.random.default_rng(seed).random(shape, dtype=np.float32) * 2 - 1
    return f32_to_bf16_bits(r * np.float32(scale))


@pytest.mark.parametrize(
    "n_out,k,t",
    [(256, 256, 16), (1376, 256, 40), (768, 688, 8), (4096, 4096, 160), (12288, 4096, 160), (4096, 11008, 160),
     (22016, 4096, 160), (2304, 768, 32), (1024, 512, 600), (12288, 4096, 645), (4096, 4096, 1280),
     (2048, 1024, 512), (5120, 13824, 1280)],  # T > 256 with an even tile count: CTA pairs (cta_group::2)
)
def test_gemm_partial_matches_fp32(n_out, k, t):
    lib = _lib.load()
    wb, xb = _rand_bf16((n_out, k), 1, 0.05), _rand_bf16((t, k), 2)
    mp, grid, bn = _info(n_out, k, t, 0)
    w, x = DeviceBuffer.from_array(wb), DeviceBuffer.from_array(xb)
    part = DeviceBuffer(4 * mp * t * n_out)
    _lib.check(lib.spin_gemm(None, w.ptr, x.ptr, n_out, k, t, 0, part.ptr, None, None, None))
    got = part.download(np.float32, (mp, t, n_out)).sum(0, dtype=np.float32)
    ref = bf16_bits_to_f32(xb).reshape(t, k) @ bf16_bits_to_f32(wb).reshape(n_out, k).T
    err = float(np.abs(got - ref).max())
    scale = float(np.abs(ref).max())
    assert err <= 1e-4 * scale + 1e-5, f"max err {err} (scale {scale}, pieces {mp}, grid {grid}, bn {bn})"


@pytest.mark.parametrize("n_out,k,t", [(4096, 256, 40), (32000, 4096, 160), (1000, 128, 5), (2048, 256, 520)])
def test_gemm_argmax_matches_fp32(n_out, k, t):
    lib = _lib.load()
    wb, xb = _rand_bf16((n_out, k), 3), _rand_bf16((t, k), 4)
    n_mt = (n_out + 127) // 128
    w, x = DeviceBuffer.from_array(wb), DeviceBuffer.from_array(xb)
    val, idx, lg = DeviceBuffer(4 * n_mt * t), DeviceBuffer(4 * n_mt * t), DeviceBuffer(4 * t * n_out)
    _lib.check(lib.spin_gemm(None, w.ptr, x.ptr, n_out, k, t, 1, None, val.ptr, idx.ptr, lg.ptr))
    val = val.download(np.float32, (n_mt, t))
    idx = idx.download(np.int32, (n_mt, t))
    logits = lg.download(np.float32, (t, n_out))
    ref = bf16_bits_to_f32(xb).reshape(t, k) @ bf16_bits_to_f32(wb).reshape(n_out, k).T
    assert np.abs(logits - ref).max() <= 1e-4 * np.abs(ref).max()
    # per-tile argmax of the kernel's own logits, lowest index on ties
    tile = val.argmax(0)
    got_idx = idx[tile, np.arange(t)]
    assert np.array_equal(got_idx, logits.argmax(1).astype(np.int32))
    assert np.array_equal(val.max(0), logits.max(1))
