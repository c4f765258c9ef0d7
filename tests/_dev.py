"""Torch-free helpers for the kernel-level GPU tests: bf16 <-> fp32 in numpy
(round to nearest even, like __float2bfloat16_rn) and device buffers owned by
libspin.so (paper_2503_15921_b200._lib.DeviceBuffer)."""
import numpy as np

from paper_2503_15921_b200._lib import DeviceBuffer  # noqa: F401


def f32_to_bf16_bits(x) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def bf16_bits_to_f32(b) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def bf16_round(x) -> np.ndarray:
    return bf16_bits_to_f32(f32_to_bf16_bits(x))
