"""ctypes binding of libspin.so, the C-ABI declared in include/spin_c.h.

The extension is the product: there is no Python or CPU fallback. If the shared
library is missing, loading raises immediately (build it with
``python -c "import __graft_entry__ as g; g.build()"`` or ``make -C
paper_2503_15921_b200/csrc``).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspin.so")

STATUS_NAMES = {
    0: "OK",
    1: "ConfigError",
    2: "CapacityError",
    3: "InputError",
    4: "SizeError",
    5: "ConsistencyError",
    6: "MetricError",
    7: "IoError",
    8: "CudaError",
}


class SpinError(RuntimeError):
    """Raised for a non-zero spin_status; `kind` is the reference exception name."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.kind = STATUS_NAMES.get(status, f"status{status}")
        super().__init__(f"{self.kind}: {message}")


class Segment(C.Structure):
    _fields_ = [
        ("request_id", C.c_int32),
        ("row", C.c_int32),
        ("col_start", C.c_int32),
        ("col_end", C.c_int32),
        ("token_offset", C.c_int32),
    ]


class ModelDesc(C.Structure):
    _fields_ = [
        ("d_model", C.c_int32),
        ("n_layers", C.c_int32),
        ("n_heads", C.c_int32),
        ("head_dim", C.c_int32),
        ("ffn", C.c_int32),
        ("vocab", C.c_int32),
        ("rope_theta", C.c_float),
        ("rms_eps", C.c_float),
        ("seed", C.c_uint64),
        ("embed_scale", C.c_float),
        ("planted_gain", C.c_float),
        ("resid_scale", C.c_float),
        ("init_scale", C.c_float),
        ("planted_domains", C.c_int32),
        ("planted_mask", C.c_uint32),
    ]


class EngineOpts(C.Structure):
    _fields_ = [
        ("device", C.c_int32),
        ("max_requests", C.c_int32),
        ("max_ctx", C.c_int32),
        ("window", C.c_int32),
        ("pack_width", C.c_int32),
        ("packing", C.c_int32),
        ("use_graphs", C.c_int32),
        ("use_pdl", C.c_int32),
        ("debug_logits", C.c_int32),
    ]


class VerifyStats(C.Structure):
    _fields_ = [("us", C.c_double), ("query_rows", C.c_int64), ("real_rows", C.c_int64), ("kv_tokens", C.c_int64),
                ("target_tokens", C.POINTER(C.c_int32))]


class ServeReport(C.Structure):
    _fields_ = [("device_ms", C.c_double), ("wall_ms", C.c_double), ("tokens", C.c_int64), ("served", C.c_int64),
                ("explore_slots", C.c_int32), ("epochs", C.c_int32), ("switch_ms", C.c_double),
                ("switch_tokens", C.c_int64)]


class RoundOut(C.Structure):
    _fields_ = [
        ("accepted", C.POINTER(C.c_int32)),
        ("bonus_token", C.POINTER(C.c_int32)),
        ("committed", C.POINTER(C.c_int32)),
        ("drafts", C.POINTER(C.c_int32)),
        ("target_tokens", C.POINTER(C.c_int32)),
        ("draft_ms", C.c_float),
        ("verify_ms", C.c_float),
        ("round_ms", C.c_float),
        ("switch_ms", C.c_float),
        ("switch_tokens", C.c_int32),
        ("spec_end_ms", C.c_float * 8),
        ("switch_tokens_per_request", C.POINTER(C.c_int32)),
    ]


_lib = None

P_I32 = C.POINTER(C.c_int32)
P_I64 = C.POINTER(C.c_int64)
P_F32 = C.POINTER(C.c_float)
P_F64 = C.POINTER(C.c_double)

# name -> argtypes (restype is always spin_status / int)
_SIGNATURES = {
    "spin_pack": [P_I32, C.c_int32, C.c_int32, P_I32, P_I32, C.POINTER(Segment), C.c_int32, P_I32, P_I64, P_I32],
    "spin_naive_padding": [P_I32, C.c_int32, P_I64],
    "spin_verify_batch_cost": [P_I32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, P_I64, P_I64],
    "spin_decomposed_attention": [C.c_int32, C.c_int32, P_I32, P_I32, P_F64, P_F64, P_F64, C.POINTER(Segment),
                                  C.c_int32, C.c_int32, C.c_int32, P_I32, P_F64],
    "spin_reference_attention": [C.c_int32, C.c_int32, C.c_int32, P_F64, P_F64, P_F64, P_F64],
    "spin_ctx_create": [C.POINTER(ModelDesc), C.POINTER(ModelDesc), C.c_int32, C.POINTER(EngineOpts),
                        C.POINTER(C.c_void_p)],
    "spin_ctx_destroy": [C.c_void_p],
    "spin_prefill": [C.c_void_p, C.c_int32, P_I32, P_I32, P_I32],
    "spin_round": [C.c_void_p, C.c_int32, P_I32, P_I32, C.POINTER(RoundOut)],
    "spin_round_prewarm": [C.c_void_p, C.c_int32, P_I32, P_I32, P_I32, C.POINTER(RoundOut)],
    "spin_set_micro_batches": [C.c_void_p, P_I32, C.c_int32],
    "spin_get_micro_batches": [C.c_void_p, P_I32, C.c_int32],
    "spin_tune_micro_batches": [C.c_void_p, C.c_int32, P_I32, P_I32, C.c_int32, C.c_int32, C.c_double, P_I32, P_F64,
                                C.c_int32, P_I32],
    "spin_run_rounds": [C.c_void_p, C.c_int32, P_I32, P_I32, C.c_int32, P_I64, P_F32],
    "spin_read_tokens": [C.c_void_p, C.c_int32, P_I32, C.c_int32, P_I32],
    "spin_read_logits": [C.c_void_p, P_F32, C.c_int64, P_I32],
    "spin_switch_ssm": [C.c_void_p, C.c_int32, P_I32, P_I32],
    "spin_profile_round": [C.c_void_p, C.c_int32, P_I32, P_I32, P_F64, P_F64, P_I64],
    "spin_round_launches": [C.c_void_p, C.c_int32, P_I32, P_I32, P_I64],
    "spin_kernel_bench": [C.c_void_p, C.c_int32, C.c_int32, P_F64, P_F64],
    "spin_attention": [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                       C.c_void_p, C.c_void_p, C.c_int32, P_I32, P_I32, P_I32, C.c_int32, C.c_void_p],
    "spin_attention_ex": [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                          C.c_void_p, C.c_void_p, C.c_int32, P_I32, P_I32, P_I32, C.c_int32, C.c_float, C.c_int32,
                          C.c_void_p],
    "spin_last_round_trace": [C.c_void_p, P_F32, C.c_int32],
    "spin_verify_bench": [C.c_void_p, C.c_int32, P_I32, P_I32, P_I32, C.c_int32, C.c_int32, C.c_void_p],
    "spin_gemm_info": [C.c_int32, C.c_int32, C.c_int32, C.c_int32, P_I32, P_I32, P_I32],
    "spin_gemm_bench": [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_double)],
    "spin_pack_device": [P_I32, C.c_int32, C.c_int32, P_I32, P_I32, C.POINTER(Segment), C.c_int32, P_I32, P_I64,
                         P_I32],
    "spin_device_count": [P_I32],
    "spin_comm_unique_id": [C.c_int32, C.c_void_p],
    "spin_comm_create": [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.POINTER(C.c_void_p)],
    "spin_comm_destroy": [C.c_void_p],
    "spin_comm_info": [C.c_void_p, P_I32, P_I32, P_I32],
    "spin_stats_allgather": [C.c_void_p, P_F64, P_F64, C.c_int32, C.c_int32],
    "spin_comm_allreduce": [C.c_void_p, P_F64, C.c_int32, C.c_int32],
    "spin_comm_barrier": [C.c_void_p],
    "spin_lbss_create": [C.c_int32, C.c_int32, P_I32, C.c_int32, C.c_int32, C.c_uint64, C.POINTER(C.c_void_p)],
    "spin_lbss_destroy": [C.c_void_p],
    "spin_lbss_next": [C.c_void_p, P_I32, P_I32, P_I32, P_I32],
    "spin_lbss_observe": [C.c_void_p, C.c_int32, C.c_int32, C.c_double],
    "spin_lbss_rows": [C.c_void_p, P_F64, C.c_int32],
    "spin_lbss_plan": [C.c_void_p, P_I32],
    "spin_lbss_peek": [C.c_void_p, P_I32],
    "spin_lbss_serve": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, P_I32, C.c_int32, C.c_int32,
                        C.c_int32, C.c_void_p, P_I32],
    "spin_device_alloc": [C.c_int32, C.c_size_t, C.POINTER(C.c_void_p)],
    "spin_device_free": [C.c_void_p],
    "spin_memcpy": [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int32],
    "spin_gemm": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                  C.c_void_p, C.c_void_p, C.c_void_p],
}


def load() -> C.CDLL:
    """Loads libspin.so once; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libspin.so not built at {LIB_PATH}; run `make -C paper_2503_15921_b200/csrc`")
    lib = C.CDLL(LIB_PATH)
    lib.spin_last_error.restype = C.c_char_p
    lib.spin_abi_version.restype = C.c_int
    for name, argtypes in _SIGNATURES.items():
        if not hasattr(lib, name):  # reported by tests/test_abi.py
            continue
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = C.c_int
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != 0:
        raise SpinError(status, load().spin_last_error().decode())


def exported_symbols() -> list[str]:
    return ["spin_abi_version", "spin_last_error", *_SIGNATURES.keys()]


def device_count() -> int:
    """CUDA devices visible to libspin.so (0 when there is no driver or device)."""
    n = C.c_int32(0)
    check(load().spin_device_count(C.byref(n)))
    return n.value


class DeviceBuffer:
    """A zero-filled device allocation owned by libspin.so (no framework needed)."""

    def __init__(self, nbytes: int, device: int = 0):
        self.nbytes = int(nbytes)
        p = C.c_void_p()
        check(load().spin_device_alloc(device, self.nbytes, C.byref(p)))
        self.ptr = p.value

    @classmethod
    def from_array(cls, a, device: int = 0) -> "DeviceBuffer":
        import numpy as np

        a = np.ascontiguousarray(a)
        buf = cls(a.nbytes, device)
        buf.upload(a)
        return buf

    def upload(self, a) -> None:
        import numpy as np

        a = np.ascontiguousarray(a)
        assert a.nbytes <= self.nbytes
        check(load().spin_memcpy(self.ptr, a.ctypes.data, a.nbytes, 1))

    def download(self, dtype, shape):
        import numpy as np

        out = np.empty(shape, dtype=dtype)
        assert out.nbytes <= self.nbytes
        check(load().spin_memcpy(out.ctypes.data, self.ptr, out.nbytes, 2))
        return out

    def free(self) -> None:
        if self.ptr:
            check(load().spin_device_free(self.ptr))
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
