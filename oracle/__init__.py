"""ctypes loaders for the CPU oracle (libspin_oracle.so) and the reference build
(_ref/libspecsim_ref.so). TEST INFRASTRUCTURE ONLY: imported by tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline / reference arm, never by
the product package."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libspin_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspecsim_ref.so")
REF_SRC = "/root/reference/proj/core/src"

_oracle = None
_ref = None


class SoModelDesc(C.Structure):
    _fields_ = [
        ("d_model", C.c_int32), ("n_layers", C.c_int32), ("n_heads", C.c_int32), ("head_dim", C.c_int32),
        ("ffn", C.c_int32), ("vocab", C.c_int32), ("rope_theta", C.c_float), ("rms_eps", C.c_float),
        ("seed", C.c_uint64), ("embed_scale", C.c_float), ("planted_gain", C.c_float),
        ("resid_scale", C.c_float), ("init_scale", C.c_float), ("planted_domains", C.c_int32),
        ("planted_mask", C.c_uint32),
    ]


def build(ref: bool | None = None) -> None:
    """Compiles the oracle (and, when the reference sources exist, oracle/_ref)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def load_oracle() -> C.CDLL:
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        lib = C.CDLL(ORACLE_SO)
        lib.so_splitmix64.restype = C.c_uint64
        lib.so_splitmix64.argtypes = [C.c_uint64]
        lib.so_mix_seed.restype = C.c_uint64
        lib.so_mix_seed.argtypes = [C.c_uint64] * 4
        lib.so_rng_next.restype = C.c_uint64
        lib.so_rng_unit.restype = C.c_double
        lib.so_rng_uniform.restype = C.c_double
        lib.so_rng_uniform.argtypes = [C.c_void_p, C.c_double, C.c_double]
        lib.so_rng_uniform_int.restype = C.c_longlong
        lib.so_rng_uniform_int.argtypes = [C.c_void_p, C.c_longlong, C.c_longlong]
        lib.so_rng_init.argtypes = [C.c_void_p, C.c_uint64]
        lib.so_make_toy_input.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                          C.c_void_p]
        lib.so_expected_accepted_prefix.restype = C.c_double
        lib.so_expected_accepted_prefix.argtypes = [C.c_double, C.c_int]
        lib.so_sample_accepted_prefix.argtypes = [C.c_double, C.c_int, C.c_void_p]
        lib.so_weight_bits.restype = C.c_uint16
        lib.so_weight_bits.argtypes = [C.POINTER(SoModelDesc), C.c_int, C.c_int, C.c_int64, C.c_int64]
        lib.so_planted_next.argtypes = [C.POINTER(SoModelDesc), C.c_int]
        lib.so_engine_create.restype = C.c_void_p
        lib.so_engine_create.argtypes = [C.POINTER(SoModelDesc), C.POINTER(SoModelDesc), C.c_int, C.c_int, C.c_int,
                                         C.c_int, C.c_int]
        lib.so_engine_destroy.argtypes = [C.c_void_p]
        lib.so_engine_prefill.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.so_engine_round.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.so_engine_switch.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        lib.so_engine_read_tokens.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p]
        lib.so_set_gemm_lanes.argtypes = [C.c_int]
        lib.so_engine_set_gap_outputs.argtypes = [C.c_void_p, C.c_void_p]
        lib.so_engine_set_hints.argtypes = [C.c_void_p, C.c_void_p, C.c_float]
        lib.so_engine_forced_count.restype = C.c_long
        lib.so_engine_forced_deficit.restype = C.c_float
        lib.so_engine_verify_ragged.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                C.c_void_p, C.c_void_p]
        lib.so_engine_fake_context.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_uint64]
        lib.so_engine_last_timing.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        lib.so_debug_layer.argtypes = [C.c_int, C.c_void_p, C.c_int]
        lib.so_debug_inner.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int]
        lib.so_engine_verify_seconds.restype = C.c_double
        lib.so_engine_verify_seconds.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO) or os.path.isdir(REF_SRC)


def load_ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build(ref=True)
        lib = C.CDLL(REF_SO)
        lib.ref_mix_seed.restype = C.c_ulonglong
        lib.ref_mix_seed.argtypes = [C.c_ulonglong] * 4
        lib.ref_rng_draws.argtypes = [C.c_ulonglong, C.c_int, C.c_longlong, C.c_longlong, C.c_int, C.c_void_p,
                                      C.c_void_p]
        lib.ref_make_toy_input.argtypes = [C.c_ulonglong, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                           C.c_void_p]
        lib.ref_expected_accepted_prefix.restype = C.c_double
        lib.ref_expected_accepted_prefix.argtypes = [C.c_double, C.c_int]
        lib.ref_sample_accepted_prefix.argtypes = [C.c_double, C.c_int, C.c_ulonglong, C.c_int, C.c_void_p]
        _ref = lib
    return _ref


def so_desc(shape) -> SoModelDesc:
    """SoModelDesc from a paper_2503_15921_b200.models.ModelShape (same fields)."""
    d = SoModelDesc()
    for f, _ in SoModelDesc._fields_:
        setattr(d, f, getattr(shape, f))
    return d


class OracleEngine:
    """CPU oracle twin of paper_2503_15921_b200.models.Engine (same round contract)."""

    def __init__(self, target, ssms, *, max_requests, max_ctx, window, threads=0):
        import numpy as np  # noqa: F401

        self.lib = load_oracle()
        self.window, self.max_ctx, self.vocab = window, max_ctx, target.vocab
        self._t = so_desc(target)
        arr = (SoModelDesc * len(ssms))(*[so_desc(s) for s in ssms])
        self._s = arr
        self.e = self.lib.so_engine_create(C.byref(self._t), arr, len(ssms), max_requests, max_ctx, window, threads)

    def close(self):
        if self.e:
            self.lib.so_engine_destroy(self.e)
            self.e = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def prefill(self, slots, prompts):
        import numpy as np

        slots = np.asarray(slots, dtype=np.int32)
        lens = np.array([len(p) for p in prompts], dtype=np.int32)
        flat = np.concatenate(prompts).astype(np.int32)
        assert self.lib.so_engine_prefill(self.e, len(slots), slots.ctypes.data, lens.ctypes.data, flat.ctypes.data) == 0

    def round(self, slots, ssm_of, want_logits=False, want_gaps=False, hints=None, tau=0.0):
        """hints: a GPU round's output dict; near-ties within tau adopt the GPU token (counted)."""
        import numpy as np

        slots = np.ascontiguousarray(slots, dtype=np.int32)
        ssm_of = np.ascontiguousarray(ssm_of, dtype=np.int32)
        n, W = len(slots), self.window
        act_rows = int((ssm_of >= 0).sum()) * (W + 1)
        dgap = np.full(n * W, np.inf, np.float32) if want_gaps else None
        tgap = np.full(max(act_rows, 1), np.inf, np.float32) if want_gaps else None
        self.lib.so_engine_set_gap_outputs(dgap.ctypes.data if want_gaps else None,
                                           tgap.ctypes.data if want_gaps else None)
        if hints is not None:
            dh = np.ascontiguousarray(hints["drafts"], dtype=np.int32).reshape(-1)
            act = np.flatnonzero(ssm_of >= 0)
            th = np.ascontiguousarray(np.asarray(hints["target"], dtype=np.int32)[act].reshape(-1))
            self._hint_keep = (dh, th)
            self.lib.so_engine_set_hints(dh.ctypes.data, th.ctypes.data, tau)
        acc, bonus, comm = np.zeros(n, np.int32), np.zeros(n, np.int32), np.zeros(n, np.int32)
        drafts, tgt = np.zeros(n * W, np.int32), np.zeros(n * (W + 1), np.int32)
        act = int((ssm_of >= 0).sum())
        logits = np.zeros(act * (W + 1) * self.vocab, np.float32) if want_logits else None
        st = self.lib.so_engine_round(self.e, n, slots.ctypes.data, ssm_of.ctypes.data, acc.ctypes.data,
                                      bonus.ctypes.data, comm.ctypes.data, drafts.ctypes.data, tgt.ctypes.data,
                                      logits.ctypes.data if want_logits else None)
        self.lib.so_engine_set_gap_outputs(None, None)
        self.lib.so_engine_set_hints(None, None, 0.0)
        assert st == 0, st
        out = {"accepted": acc, "bonus": bonus, "committed": comm, "drafts": drafts.reshape(n, W),
               "target": tgt.reshape(n, W + 1)}
        if want_gaps:
            out["draft_gap"] = dgap.reshape(n, W)
            out["target_gap"] = tgap[:act_rows]
        if want_logits:
            out["logits"] = logits.reshape(act * (W + 1), self.vocab)
        return out

    def forced(self) -> int:
        """Near-tie decisions adopted from the GPU since the last reset (process-wide)."""
        return int(self.lib.so_engine_forced_count())

    def forced_deficit(self) -> float:
        """Largest (own max logit - adopted logit) over those decisions."""
        return float(self.lib.so_engine_forced_deficit())

    def reset_forced(self) -> None:
        self.lib.so_engine_reset_forced()

    def verify_ragged(self, slots, draft_lens, drafts, hint=None, tau=0.0, want_logits=False):
        """Target argmax of every row of a ragged verification (spin_verify_bench contract)."""
        import numpy as np

        slots = np.ascontiguousarray(slots, dtype=np.int32)
        lens = np.ascontiguousarray(draft_lens, dtype=np.int32)
        dr = np.ascontiguousarray(drafts, dtype=np.int32)
        rows = int(lens.sum()) + len(lens)
        out = np.zeros(rows, np.int32)
        hv = None
        if hint is not None:
            hv = np.ascontiguousarray(hint, dtype=np.int32)
            self.lib.so_engine_set_hints(None, None, tau)
        logits = np.zeros(rows * self.vocab, np.float32) if want_logits else None
        st = self.lib.so_engine_verify_ragged(self.e, len(slots), slots.ctypes.data, lens.ctypes.data, dr.ctypes.data,
                                              hv.ctypes.data if hv is not None else None, out.ctypes.data,
                                              logits.ctypes.data if want_logits else None)
        self.lib.so_engine_set_hints(None, None, 0.0)
        assert st == 0, st
        return (out, logits.reshape(rows, self.vocab)) if want_logits else out

    def fake_context(self, slots, lens, seed: int = 2503):
        """Seeded histories + KV rows instead of a prefill forward (CPU-baseline timing only)."""
        import numpy as np

        slots = np.ascontiguousarray(slots, dtype=np.int32)
        lens = np.ascontiguousarray(lens, dtype=np.int32)
        assert self.lib.so_engine_fake_context(self.e, len(slots), slots.ctypes.data, lens.ctypes.data, seed) == 0

    def last_timing(self):
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        self.lib.so_engine_last_timing(C.byref(a), C.byref(b), C.byref(c))
        return a.value, b.value, c.value

    def tokens(self, slot):
        import numpy as np

        buf = np.zeros(self.max_ctx, np.int32)
        n = C.c_int()
        assert self.lib.so_engine_read_tokens(self.e, slot, buf.ctypes.data, self.max_ctx, C.byref(n)) == 0
        return buf[: n.value].copy()

    def verify_seconds(self, slots):
        import numpy as np

        slots = np.ascontiguousarray(slots, dtype=np.int32)
        return self.lib.so_engine_verify_seconds(self.e, len(slots), slots.ctypes.data)
