"""Model shapes of BASELINE.json's configs and a thin Python wrapper over the
C-ABI engine (include/spin_c.h) used by the tests and bench.py.

Weights are synthetic (seeded, random-init) with a planted next-token map so
that independent random SSMs still agree with the target at controllable,
heterogeneous rates.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, asdict, replace

import numpy as np

from . import _lib


@dataclass(frozen=True)
class ModelShape:
    name: str
    d_model: int
    n_layers: int
    n_heads: int
    head_dim: int
    ffn: int
    vocab: int
    seed: int
    planted_gain: float = 12.0
    resid_scale: float = 0.5
    init_scale: float = 1.0
    embed_scale: float = 1.0
    rope_theta: float = 10000.0
    rms_eps: float = 1e-5
    planted_domains: int = 0  # token domains of the planted map (0/1: one); pi keeps each domain
    planted_mask: int = 0     # domains whose lm_head rows carry the planted term (0: all)

    def desc(self) -> _lib.ModelDesc:
        d = _lib.ModelDesc()
        for f in ("d_model", "n_layers", "n_heads", "head_dim", "ffn", "vocab", "rope_theta", "rms_eps", "seed",
                  "embed_scale", "planted_gain", "resid_scale", "init_scale", "planted_domains", "planted_mask"):
            setattr(d, f, getattr(self, f))
        return d

    def params(self) -> int:
        D, F, V = self.d_model, self.ffn, self.vocab
        return 2 * V * D + self.n_layers * (4 * D * D + 3 * D * F)

    def block_params(self) -> int:
        D, F = self.d_model, self.ffn
        return self.n_layers * (4 * D * D + 3 * D * F)


# ---- BASELINE.json configs
TINY_TARGET = ModelShape("tiny-target", 256, 4, 4, 64, 688, 4096, seed=2503, planted_gain=9.0, resid_scale=0.15)
TINY_SSMS = (
    ModelShape("tiny-ssm-a", 128, 1, 2, 64, 344, 4096, seed=2504, planted_gain=7.0, resid_scale=1.2),
    ModelShape("tiny-ssm-b", 256, 2, 4, 64, 688, 4096, seed=2505, planted_gain=8.0, resid_scale=0.8),
)
LLAMA_7B = ModelShape("llama-7b-shape", 4096, 32, 32, 128, 11008, 32000, seed=7001, planted_gain=12.0,
                      resid_scale=0.5)
LLAMA_13B = ModelShape("llama-13b-shape", 5120, 40, 40, 128, 13824, 32000, seed=13001, planted_gain=12.0,
                       resid_scale=0.5)
LLAMA_68M = ModelShape("llama-68m-shape", 768, 2, 12, 64, 3072, 32000, seed=68001, planted_gain=9.0,
                       resid_scale=1.0)
LLAMA_160M = ModelShape("llama-160m-shape", 768, 12, 12, 64, 3072, 32000, seed=160001, planted_gain=10.0,
                        resid_scale=0.7)
LLAMA_160M_B = ModelShape("llama-160m-shape-b", 768, 12, 12, 64, 3072, 32000, seed=160002, planted_gain=8.0,
                          resid_scale=0.9)


# ---- config 4 with per-request heterogeneity: 4 token domains; the target plants every
# domain, each SSM only some, so the best SSM depends on the request (its domain): the
# 68M SSM is cheap but only knows domain 0, the 160M knows 0-2, the 160M-b knows 2-3.
# The target's planted gain is raised to 20 so that its greedy continuation follows the map
# (at 12 the 40-layer target leaves the prompt's domain within a few tokens: 35% of generated
# tokens stay in it; at 20, 100% -- tools/scratch/domain_probe.py), and the 160M-b SSM gets the
# 160M's gain so it is as good on its own domains.
C4_DOMAINS = 4
LLAMA_13B_DOM = replace(LLAMA_13B, name="llama-13b-shape-dom4", planted_domains=C4_DOMAINS, planted_gain=20.0)
LLAMA_68M_DOM = replace(LLAMA_68M, name="llama-68m-shape-d0", planted_domains=C4_DOMAINS, planted_mask=0b0001)
LLAMA_160M_DOM = replace(LLAMA_160M, name="llama-160m-shape-d012", planted_domains=C4_DOMAINS, planted_mask=0b0111)
LLAMA_160M_B_DOM = replace(LLAMA_160M_B, name="llama-160m-shape-b-d23", planted_domains=C4_DOMAINS,
                           planted_mask=0b1100, planted_gain=10.0, resid_scale=0.7)


def domain_prompts(n: int, lo: int, hi: int, vocab: int, n_domains: int, seed: int) -> list[np.ndarray]:
    """Prompt lengths U[lo, hi]; request i's tokens U over its domain i % n_domains
    (vocab / n_domains contiguous ids), which the planted map keeps it in."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(lo, hi + 1, n)
    size = vocab // n_domains
    return [(size * (i % n_domains) + rng.integers(0, size, int(L))).astype(np.int32) for i, L in enumerate(lens)]


def synthetic_prompts(n: int, lo: int, hi: int, vocab: int, seed: int) -> list[np.ndarray]:
    """Prompt lengths U[lo, hi], token ids U[0, vocab) from a seeded generator."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(lo, hi + 1, n)
    return [rng.integers(0, vocab, int(L)).astype(np.int32) for L in lens]


def _p(a: np.ndarray, t=C.c_int32):
    return a.ctypes.data_as(C.POINTER(t))


class Engine:
    """One spin_ctx: target + SSMs on one GPU."""

    def __init__(self, target: ModelShape, ssms, *, max_requests: int, max_ctx: int, window: int, device: int = 0,
                 pack_width: int = 0, packing: bool = True, use_graphs: bool = True, use_pdl: bool = True,
                 debug_logits: bool = False):
        self.lib = _lib.load()
        self.target, self.ssms, self.window = target, tuple(ssms), window
        self.max_requests, self.max_ctx = max_requests, max_ctx
        opts = _lib.EngineOpts(device, max_requests, max_ctx, window, pack_width, int(packing), int(use_graphs),
                               int(use_pdl), int(debug_logits))
        descs = (_lib.ModelDesc * len(self.ssms))(*[s.desc() for s in self.ssms])
        td = target.desc()
        ctx = C.c_void_p()
        _lib.check(self.lib.spin_ctx_create(C.byref(td), descs, len(self.ssms), C.byref(opts), C.byref(ctx)))
        self.ctx = ctx

    def close(self):
        if self.ctx:
            _lib.check(self.lib.spin_ctx_destroy(self.ctx))
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def prefill(self, slots, prompts):
        slots = np.asarray(slots, dtype=np.int32)
        lens = np.array([len(p) for p in prompts], dtype=np.int32)
        flat = np.concatenate(prompts).astype(np.int32)
        _lib.check(self.lib.spin_prefill(self.ctx, len(slots), _p(slots), _p(lens), _p(flat)))

    def round(self, slots, ssm_of, prewarm=None):
        """One speculation + verification slot (spin_round / spin_round_prewarm).
        prewarm[i] (or -1): SSM whose KV is warmed for request i while the round runs."""
        slots = np.ascontiguousarray(slots, dtype=np.int32)
        ssm_of = np.ascontiguousarray(ssm_of, dtype=np.int32)
        n, W = len(slots), self.window
        acc = np.zeros(n, np.int32)
        bonus = np.zeros(n, np.int32)
        comm = np.zeros(n, np.int32)
        drafts = np.zeros(n * W, np.int32)
        tgt = np.zeros(n * (W + 1), np.int32)
        sw = np.zeros(n, np.int32)
        out = _lib.RoundOut(_p(acc), _p(bonus), _p(comm), _p(drafts), _p(tgt), 0.0, 0.0, 0.0)
        out.switch_tokens_per_request = _p(sw)
        if prewarm is None:
            _lib.check(self.lib.spin_round(self.ctx, n, _p(slots), _p(ssm_of), C.byref(out)))
        else:
            pw = np.ascontiguousarray(prewarm, dtype=np.int32)
            _lib.check(self.lib.spin_round_prewarm(self.ctx, n, _p(slots), _p(ssm_of), _p(pw), C.byref(out)))
        spec_end = np.array(out.spec_end_ms[: len(self.ssms)], np.float32)
        # per-request wall time (SlotRecord.wall_time_sec, slot_engine.cpp:145): own SSM's draft end + verify
        wall_ms = np.where(ssm_of >= 0, spec_end[np.maximum(ssm_of, 0)] + out.verify_ms, 0.0)
        return {"accepted": acc, "bonus": bonus, "committed": comm, "drafts": drafts.reshape(n, W),
                "target": tgt.reshape(n, W + 1), "draft_ms": out.draft_ms, "verify_ms": out.verify_ms,
                "round_ms": out.round_ms, "switch_ms": out.switch_ms, "switch_tokens": out.switch_tokens,
                "switch_tokens_per_request": sw, "spec_end_ms": spec_end, "wall_ms": wall_ms}

    def run_rounds(self, slots, ssm_of, rounds: int):
        slots = np.ascontiguousarray(slots, dtype=np.int32)
        ssm_of = np.ascontiguousarray(ssm_of, dtype=np.int32)
        emitted = np.zeros(rounds, np.int64)
        ms = C.c_float()
        _lib.check(self.lib.spin_run_rounds(self.ctx, len(slots), _p(slots), _p(ssm_of), rounds,
                                            emitted.ctypes.data_as(_lib.P_I64), C.byref(ms)))
        return emitted, ms.value

    def tokens(self, slot: int) -> np.ndarray:
        buf = np.zeros(self.max_ctx, np.int32)
        n = C.c_int32()
        _lib.check(self.lib.spin_read_tokens(self.ctx, slot, _p(buf), self.max_ctx, C.byref(n)))
        return buf[: n.value].copy()

    def logits(self, rows_cap: int) -> np.ndarray:
        buf = np.zeros(rows_cap * self.target.vocab, np.float32)
        rows = C.c_int32()
        _lib.check(self.lib.spin_read_logits(self.ctx, buf.ctypes.data_as(_lib.P_F32), buf.size, C.byref(rows)))
        return buf[: rows.value * self.target.vocab].reshape(rows.value, self.target.vocab)

    PROF_CLASSES = ("target_gemm", "target_lm_head", "target_attention", "target_epilogue", "ssm_gemm",
                    "ssm_lm_head", "ssm_attention", "ssm_epilogue", "meta_accept")

    def profile(self, slots, ssm_of):
        """One un-graphed round with CUDA events around each launch: {class: (ms, bytes, launches)}."""
        slots = np.ascontiguousarray(slots, dtype=np.int32)
        ssm_of = np.ascontiguousarray(ssm_of, dtype=np.int32)
        ms, by, ln = np.zeros(9), np.zeros(9), np.zeros(9, np.int64)
        _lib.check(self.lib.spin_profile_round(self.ctx, len(slots), _p(slots), _p(ssm_of), ms.ctypes.data_as(_lib.P_F64),
                                               by.ctypes.data_as(_lib.P_F64), ln.ctypes.data_as(_lib.P_I64)))
        return {k: (float(ms[i]), float(by[i]), int(ln[i])) for i, k in enumerate(self.PROF_CLASSES)}

    def launches_per_round(self, slots, ssm_of) -> int:
        slots = np.ascontiguousarray(slots, dtype=np.int32)
        ssm_of = np.ascontiguousarray(ssm_of, dtype=np.int32)
        v = C.c_int64()
        _lib.check(self.lib.spin_round_launches(self.ctx, len(slots), _p(slots), _p(ssm_of), C.byref(v)))
        return v.value

    def kernel_bench(self, kind: str, iters: int = 5):
        """(us per launch, algorithmic bytes per launch) of the target's GEMMs ("gemm") or attention ("attention")."""
        us, by = C.c_double(), C.c_double()
        _lib.check(self.lib.spin_kernel_bench(self.ctx, {"gemm": 0, "attention": 1}[kind], iters, C.byref(us),
                                              C.byref(by)))
        return us.value, by.value

    def verify_bench(self, slots, draft_lens, drafts=None, packed: bool = True, iters: int = 5):
        """Ragged-window verification step (config 3): device us per step, rows, KV tokens read,
        and the target argmax of every real query row (concatenated per request)."""
        slots = np.ascontiguousarray(slots, dtype=np.int32)
        lens = np.ascontiguousarray(draft_lens, dtype=np.int32)
        tgt = np.zeros(int(lens.sum()) + len(lens), np.int32)
        st = _lib.VerifyStats()
        st.target_tokens = tgt.ctypes.data_as(_lib.P_I32)
        dr = None
        if drafts is not None:
            dr = np.ascontiguousarray(drafts, dtype=np.int32)
        _lib.check(self.lib.spin_verify_bench(self.ctx, len(slots), _p(slots), _p(lens),
                                              _p(dr) if dr is not None else None, int(packed), iters, C.byref(st)))
        return {"us": st.us, "query_rows": st.query_rows, "real_rows": st.real_rows, "kv_tokens": st.kv_tokens,
                "target": tgt}

    def set_micro_batches(self, per_ssm):
        """Speculation/verification pipelining plan (spin_set_micro_batches); all ones = serial."""
        p = np.ascontiguousarray(per_ssm, dtype=np.int32)
        _lib.check(self.lib.spin_set_micro_batches(self.ctx, _p(p), len(p)))

    def micro_batches(self) -> np.ndarray:
        p = np.zeros(len(self.ssms), np.int32)
        _lib.check(self.lib.spin_get_micro_batches(self.ctx, _p(p), len(p)))
        return p

    def tune_micro_batches(self, slots, ssm_of, max_micro_batches=4, probe_rounds=4, threshold=0.05):
        """tune_micro_batches on measured throughput; returns (chosen plan, curve of tokens/s)."""
        slots = np.ascontiguousarray(slots, dtype=np.int32)
        ssm_of = np.ascontiguousarray(ssm_of, dtype=np.int32)
        chosen = np.zeros(len(self.ssms), np.int32)
        curve = np.zeros(16, np.float64)
        k = C.c_int32()
        _lib.check(self.lib.spin_tune_micro_batches(self.ctx, len(slots), _p(slots), _p(ssm_of), max_micro_batches,
                                                    probe_rounds, threshold, _p(chosen),
                                                    curve.ctypes.data_as(_lib.P_F64), 16, C.byref(k)))
        return chosen, curve[: k.value].tolist()

    def switch(self, slots, ssm_of):
        slots = np.ascontiguousarray(slots, dtype=np.int32)
        ssm_of = np.ascontiguousarray(ssm_of, dtype=np.int32)
        _lib.check(self.lib.spin_switch_ssm(self.ctx, len(slots), _p(slots), _p(ssm_of)))


def shape_dict(m: ModelShape) -> dict:
    return asdict(m)
