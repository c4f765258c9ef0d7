"""Runs the projection GEMM (spin_gemm, PARTIAL epilogue) on the 7B projection shapes
at T = 160 / 645 / 1280 token rows -- the config-2, config-3 (mean gamma ~8.5) and
config-5 (256 requests) verification row counts -- with device buffers from libspin.
Timed with CUDA events around `reps` back-to-back launches each (printed), and the
target of `ncu --set full --kernel-name gemm_tc_kernel` captures (tensor-pipe %)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2503_15921_b200 import _lib
from paper_2503_15921_b200._lib import DeviceBuffer

SHAPES = {"qkv": (12288, 4096), "o": (4096, 4096), "gate_up": (22016, 4096), "down": (4096, 11008)}
TS = [int(t) for t in os.environ.get("PROBE_T", "160,645,1280").split(",")]
reps = int(os.environ.get("PROBE_REPS", "1"))
lib = _lib.load()
rng = np.random.default_rng(0)
for t in TS:
    for name, (n_out, k) in SHAPES.items():
        mp, grid, bn = C.c_int32(), C.c_int32(), C.c_int32()
        _lib.check(lib.spin_gemm_info(n_out, k, t, 0, C.byref(mp), C.byref(grid), C.byref(bn)))
        w = DeviceBuffer(2 * n_out * k)
        x = DeviceBuffer.from_array((rng.integers(0, 1 << 14, (t, k))).astype(np.uint16))
        part = DeviceBuffer(4 * mp.value * t * n_out)
        for _ in range(reps):
            _lib.check(lib.spin_gemm(None, w.ptr, x.ptr, n_out, k, t, 0, part.ptr, None, None, None))
        print(f"T={t} {name} {n_out}x{k}: pieces {mp.value} grid {grid.value} bn {bn.value} "
              f"flops {2.0 * t * n_out * k:.3e}", flush=True)
        for b in (w, x, part):
            b.free()
