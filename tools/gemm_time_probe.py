"""Times the projection GEMM (PARTIAL epilogue) on the 7B / 13B projection shapes at
T = 160 / 645 / 1280 token rows through spin_gemm_bench (production plan, launches
back to back in one CUDA graph with PDL, CUDA events). Environment switches of
gemm_plan (e.g. SPIN_GEMM_PAIR_MIN_T) select the variant; PROBE_TAG labels the lines."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_15921_b200 import _lib

SHAPES = {"qkv": (12288, 4096), "o": (4096, 4096), "gate_up": (22016, 4096), "down": (4096, 11008)}
TS = [int(t) for t in os.environ.get("PROBE_T", "160,645,1280").split(",")]
iters = int(os.environ.get("PROBE_ITERS", "20"))
tag = os.environ.get("PROBE_TAG", "")
lib = _lib.load()
for t in TS:
    for name, (n_out, k) in SHAPES.items():
        mp, grid, bn = C.c_int32(), C.c_int32(), C.c_int32()
        _lib.check(lib.spin_gemm_info(n_out, k, t, 0, C.byref(mp), C.byref(grid), C.byref(bn)))
        us = C.c_double()
        _lib.check(lib.spin_gemm_bench(n_out, k, t, 0, iters, C.byref(us)))
        us = us.value
        fl = 2.0 * t * n_out * k
        by = 2.0 * n_out * k + 2.0 * t * k
        print(f"{tag} T={t:5d} {name:8s} grid {grid.value:3d} bn {bn.value:3d} pieces {mp.value}: {us:7.1f} us "
              f"{fl / us / 1e6:6.0f} TFLOP/s {by / us / 1e3:6.0f} GB/s", flush=True)
