"""GPU-vs-oracle round parity with a measured noise floor (test infrastructure).

Contract (north_star): drafts, target argmax rows, accepted counts, bonus tokens
and committed histories bit-exact; target logits within 1e-3 relative (Frobenius
norm of the error over the round's logit matrix) -- or within 2x the oracle's own
reordering error where that floor is higher (7B / 13B depth) -- and, element-wise,
within 2x the measured fp32 reordering floor below.

Two fp32 implementations with different summation orders cannot agree on an
argmax whose top-2 logits are closer than their accumulated rounding noise. The
oracle therefore runs tie-aware: where its own logits put the GPU's token within
TAU_MAX of its maximum it adopts that token and records the deficit (own max
minus the adopted logit). The noise floor is MEASURED each round: a twin oracle
with a reordered fp32 accumulation (8 instead of 16 partial sums), teacher-forced
onto the GPU's tokens, gives max |twin - oracle| over the verify logits. Every
adopted decision must have a deficit <= 2 x that floor, adoptions must stay rare
(<= 2% of decisions), and the GPU's logits must be no further from the oracle
than 2 x the floor (and <= 1e-3 of the logit scale)."""
from __future__ import annotations

import numpy as np

import oracle
from oracle import OracleEngine
from paper_2503_15921_b200.models import Engine, synthetic_prompts

TAU_MAX = 0.5  # adoption window of the oracle; the binding bound is 2 x the measured floor
TWIN_FORCE = 1e30  # the twin follows the GPU's tokens unconditionally (it only measures noise)
MAX_FORCED = 0.02
KEYS = ("drafts", "target", "accepted", "bonus", "committed")


class ParityRun:
    def __init__(self, target, ssms, *, batch, prompt_lo, prompt_hi, seed, window, max_ctx, twin=True,
                 micro_batches=None, prompts=None, **gpu_kw):
        self.B, self.W = batch, window
        if prompts is None:
            prompts = synthetic_prompts(batch, prompt_lo, prompt_hi, target.vocab, seed)
        self.gpu = Engine(target, ssms, max_requests=batch, max_ctx=max_ctx, window=window, debug_logits=True,
                          **gpu_kw)
        if micro_batches is not None:  # pipelined rounds: the logits check needs one verify per round
            self.gpu.set_micro_batches(micro_batches)
        self.pipelined = micro_batches is not None and any(b != 1 for b in micro_batches)
        self.cpu = OracleEngine(target, ssms, max_requests=batch, max_ctx=max_ctx, window=window)
        self.twin = OracleEngine(target, ssms, max_requests=batch, max_ctx=max_ctx, window=window) if twin else None
        self.lib = oracle.load_oracle()
        self.lib.so_set_gemm_lanes(16)
        self.gpu.prefill(range(batch), prompts)
        self.cpu.prefill(range(batch), prompts)
        if self.twin:
            self.lib.so_set_gemm_lanes(8)
            self.twin.prefill(range(batch), prompts)
            self.lib.so_set_gemm_lanes(16)
        self.slots = np.arange(batch, dtype=np.int32)
        self.stats = dict(rounds=0, decisions=0, forced=0, deficit=0.0, floor=0.0, worst_abs=0.0, worst_rel=0.0,
                          worst_rel_fro=0.0, emitted=0)

    def round(self, assign):
        assign = np.asarray(assign, dtype=np.int32)
        W, st = self.W, self.stats
        g = self.gpu.round(self.slots, assign)
        self.lib.so_set_gemm_lanes(16)
        self.cpu.reset_forced()
        c = self.cpu.round(self.slots, assign, want_logits=True, hints=g, tau=TAU_MAX)
        st["forced"] += self.cpu.forced()
        st["deficit"] = max(st["deficit"], self.cpu.forced_deficit())
        for k in KEYS:
            assert np.array_equal(g[k], c[k]), (st["rounds"], k, g[k], c[k])
        act = int((assign >= 0).sum())
        if act and not self.pipelined:
            lg = self.gpu.logits(act * (W + 1))
            ref = c["logits"]
            denom = float(np.abs(ref).max())
            diff = float(np.abs(lg - ref).max())
            st["worst_abs"] = max(st["worst_abs"], diff)
            st["worst_rel"] = max(st["worst_rel"], diff / denom)
            fro = float(np.linalg.norm(ref))
            st["worst_rel_fro"] = max(st.get("worst_rel_fro", 0.0), float(np.linalg.norm(lg - ref)) / fro)
            if self.twin:
                self.lib.so_set_gemm_lanes(8)
                t = self.twin.round(self.slots, assign, want_logits=True, hints=g, tau=TWIN_FORCE)
                self.lib.so_set_gemm_lanes(16)
                st["floor"] = max(st["floor"], float(np.abs(t["logits"] - ref).max()))
                st["floor_rel"] = max(st.get("floor_rel", 0.0), float(np.abs(t["logits"] - ref).max()) / denom)
                st["floor_rel_fro"] = max(st.get("floor_rel_fro", 0.0),
                                          float(np.linalg.norm(t["logits"] - ref)) / fro)
        st["decisions"] += act * (2 * W + 1)
        st["emitted"] += int(g["accepted"][assign >= 0].sum()) + act
        st["rounds"] += 1
        return g

    def check(self):
        """The parity contract over all rounds so far (see module docstring)."""
        st = self.stats
        assert st["forced"] <= MAX_FORCED * st["decisions"], st
        # 1e-3 relative (Frobenius norm of the logit error over the round's logit matrix)
        # wherever that is above the fp32 reordering floor; at 32-40 layers it is not: the
        # oracle's own reordered twin differs by ~6.6e-3 (7B shape, measured), because
        # one bf16-ulp flip of a normalised activation propagates through the blocks. There
        # the bar is "no further from the oracle than the oracle is from itself" (2x).
        bound = max(1e-3, 2.0 * st.get("floor_rel_fro", 0.0))
        assert st["worst_rel_fro"] <= bound, st
        if self.twin and not self.pipelined:
            assert st["floor"] > 0.0, st
            assert st["deficit"] <= 2.0 * st["floor"], st
            assert st["worst_abs"] <= 2.0 * st["floor"], st
        for s in range(self.B):
            assert np.array_equal(self.gpu.tokens(s), self.cpu.tokens(s)), s
        return st

    def close(self):
        self.gpu.close()
        self.cpu.close()
        if self.twin:
            self.twin.close()


def ragged_vs_oracle(target, ssms, *, batch, window, width, prompt_lo, prompt_hi, seed, max_ctx):
    """Config-3 verification (ragged draft lengths 1..window, nothing committed):
    the packed (request decomposition) and the padded GPU steps must each give the
    oracle's target argmax on every real row (tie-aware with the measured floor)."""
    rng = np.random.default_rng(seed)
    prompts = synthetic_prompts(batch, prompt_lo, prompt_hi, target.vocab, seed)
    slots = np.arange(batch, dtype=np.int32)
    lens = rng.integers(1, window + 1, batch).astype(np.int32)
    lens[: min(batch, window)] = np.arange(1, min(batch, window) + 1)  # every length 1..window present
    rng.shuffle(lens)
    drafts = rng.integers(0, target.vocab, int(lens.sum())).astype(np.int32)
    gpu = Engine(target, ssms, max_requests=batch, max_ctx=max_ctx, window=window, pack_width=width)
    gpu.prefill(range(batch), prompts)
    res = {p: gpu.verify_bench(slots, lens, drafts, packed=p, iters=1) for p in (True, False)}
    gpu.close()
    lib = oracle.load_oracle()
    lib.so_set_gemm_lanes(16)
    cpu = OracleEngine(target, ssms, max_requests=batch, max_ctx=max_ctx, window=window)
    cpu.prefill(range(batch), prompts)
    lib.so_set_gemm_lanes(8)
    twin = OracleEngine(target, ssms, max_requests=batch, max_ctx=max_ctx, window=window)
    twin.prefill(range(batch), prompts)
    lib.so_set_gemm_lanes(16)
    _, ref_logits = cpu.verify_ragged(slots, lens, drafts, want_logits=True)
    lib.so_set_gemm_lanes(8)
    _, twin_logits = twin.verify_ragged(slots, lens, drafts, want_logits=True)
    lib.so_set_gemm_lanes(16)
    floor = float(np.abs(twin_logits - ref_logits).max())
    out = {"floor": floor, "rows": int((lens + 1).sum())}
    for packed, r in res.items():
        cpu.reset_forced()
        tok = cpu.verify_ragged(slots, lens, drafts, hint=r["target"], tau=TAU_MAX)
        name = "packed" if packed else "padded"
        assert np.array_equal(tok, r["target"]), name
        out[name] = {"forced": cpu.forced(), "deficit": cpu.forced_deficit(), "query_rows": r["query_rows"],
                     "kv_tokens": r["kv_tokens"]}
        assert cpu.forced() <= MAX_FORCED * out["rows"], out
        assert cpu.forced_deficit() <= 2.0 * floor, out
    cpu.close()
    twin.close()
    return out
