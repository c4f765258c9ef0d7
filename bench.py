"""Benchmark of the B200 Spin verification path (BASELINE.json config 2).

Workload ("step" = one speculation + verification round, SlotEngine::run_slot):
LLaMA-7B-shaped target verifying drafts from LLaMA-68M- and LLaMA-160M-shaped
SSMs (half the batch each), batch 32 per GPU, gamma = 4, prompts U[128, 512],
synthetic random-init weights with a planted next-token map.

  value  accepted tokens/s with everything resident in HBM: spin_run_rounds,
         rounds back to back on the device, CUDA-event timed, max over ranks.
  e2e    the same metric through the public per-slot C-ABI call spin_round
         (host buffers; H2D of the assignment and D2H of the outcome inside
         every step) plus, at N > 1, the per-step all-gather of per-(request, SSM)
         acceptance statistics (spin_stats_allgather over NCCL); wall-clock
         timed, max over ranks.

Multi-GPU: one process per GPU. Under torchrun the ranks come from the
environment; `python bench.py --gpus N` without WORLD_SIZE spawns the N ranks
itself. Collectives go through libspin's communicator (NCCL); torch only hands rank
0's NCCL id to the other ranks when torchrun launched them.

`--impl reference` times the CPU implementation of the same path on the host
cores (the oracle port of the reference's semantics: the reference itself only
simulates this path) on a bounded sample of the workload, and the reference's
own single-threaded hot-path functions (pack, verify_batch_cost,
decomposed_attention, SlotEngine::run_slot), and prints the same JSON line.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "accepted tokens/sec at batch 32, gamma=4 (verify-step us and % of roofline in roofline/config)"
UNIT = "tokens/s"
BATCH, WINDOW = 32, 4
PROMPT_LO, PROMPT_HI = 128, 512
SEED = 2503


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms while running."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, peak_sm_mhz=None):
        rows = []
        try:
            with open(self.path) as f:
                for line in f:
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": peak_sm_mhz, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else peak_sm_mhz,
                "reasons": reasons, "samples": len(rows)}


def path_roofline_us(target, committed, window, hbm_gbs, tflops):
    """algorithmic bytes / flops of one verify step."""
    D, F, V, L = target.d_model, target.ffn, target.vocab, target.n_layers
    n = len(committed)
    T = n * (window + 1)
    P_blk = L * (4 * D * D + 3 * D * F)
    C = sum(int(c) - 1 for c in committed)  # cached tokens read
    bytes_ = 2 * (P_blk + V * D) + 4 * L * D * C + 4 * L * D * T + 2 * T * D
    flops = 2 * T * (P_blk + V * D) + 4 * L * D * sum((window + 1) * (int(c) + window) for c in committed)
    t_hbm = bytes_ / (hbm_gbs * 1e9) * 1e6
    t_tc = flops / (tflops * 1e12) * 1e6
    return max(t_hbm, t_tc), bytes_, flops


# ---------------------------------------------------------------- ranks and collectives
class Ranks:
    """rank / world / device, and libspin's communicator for N > 1: NCCL (ncclAllGather of
    the stats rows); the TCP transport when SPIN_COMM=tcp or when NCCL cannot initialise
    (same gather semantics; the gathered rows are host data either way).
    SPIN_BENCH_SHARE_DEVICE=1 puts every rank on device 0 (functional runs of the N > 1
    path on a one-GPU box; NCCL refuses two ranks on one device, so it implies TCP)."""

    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.shared = os.environ.get("SPIN_BENCH_SHARE_DEVICE", "0") == "1"
        self.device = 0 if self.shared else self.local
        self.comm = None
        self.backend = None
        if self.world > 1:
            from paper_2503_15921_b200 import _lib, dist

            want = "tcp" if self.shared or os.environ.get("SPIN_COMM", "nccl") == "tcp" else "nccl"
            ids = os.environ.get("SPIN_COMM_ID")
            if ids is None:  # launched by torchrun: rank 0's ids travel over torch's CPU store
                import torch.distributed as tdist

                tdist.init_process_group("gloo")
                obj = [None]
                if self.rank == 0:
                    nccl = dist.unique_id(dist.NCCL).hex() if want == "nccl" else ""
                    obj = [nccl + ":" + dist.unique_id(dist.TCP).hex()]
                tdist.broadcast_object_list(obj, src=0)
                ids = obj[0]
                tdist.destroy_process_group()
            nccl_id, tcp_id = ids.split(":")
            if want == "nccl" and nccl_id:
                try:
                    self.comm = dist.Comm(dist.NCCL, self.rank, self.world, bytes.fromhex(nccl_id), self.device)
                    self.backend = "nccl"
                except _lib.SpinError as e:
                    print(f"rank {self.rank}: NCCL communicator failed ({e}); using the TCP transport",
                          file=sys.stderr, flush=True)
            if self.comm is None:
                self.comm = dist.Comm(dist.TCP, self.rank, self.world, bytes.fromhex(tcp_id), self.device)
                self.backend = "tcp"

    def barrier(self):
        if self.comm is not None:
            self.comm.barrier()

    def max(self, x):
        return self.comm.max(x) if self.comm is not None else x

    def sum(self, x):
        return self.comm.sum(x) if self.comm is not None else x

    def close(self):
        if self.comm is not None:
            self.comm.close()


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` without WORLD_SIZE: one process per GPU, NCCL id from here."""
    from paper_2503_15921_b200 import dist

    nccl = "" if os.environ.get("SPIN_COMM") == "tcp" or os.environ.get("SPIN_BENCH_SHARE_DEVICE") == "1" \
        else dist.unique_id(dist.NCCL).hex()
    ids = nccl + ":" + dist.unique_id(dist.TCP).hex()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(n), LOCAL_RANK=str(r), LOCAL_WORLD_SIZE=str(n),
                   SPIN_COMM_ID=ids, MASTER_ADDR="127.0.0.1")
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), *sys.argv[1:]], env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    return max(p.wait() for p in procs)


# ---------------------------------------------------------------- CPU baseline (oracle port)
def cpu_sample(steps: int, warm: int = 1, bs: int = 4):
    """Oracle port on the host cores: config-2 rounds on a bounded sample, no extrapolation.

    Sample: the first `bs` of the 32 requests with their real config-2 context lengths
    (the KV caches of target and SSMs filled with seeded values instead of running
    the prefill forward -- a verify over a context costs the same either way), the
    full 32-layer 7B-shaped target and full-depth SSMs, greedy rounds exactly as the
    GPU path runs them. Accepted tokens / wall seconds of the rounds.
    """
    from oracle import OracleEngine
    from paper_2503_15921_b200.models import LLAMA_7B, LLAMA_68M, LLAMA_160M, synthetic_prompts

    prompts = synthetic_prompts(BATCH, PROMPT_LO, PROMPT_HI, LLAMA_7B.vocab, SEED)[:bs]
    lens = np.array([len(p) for p in prompts], np.int32)
    eng = OracleEngine(LLAMA_7B, (LLAMA_68M, LLAMA_160M), max_requests=bs,
                       max_ctx=PROMPT_HI + (WINDOW + 1) * (steps + warm + 2) + 8, window=WINDOW, threads=0)
    slots = np.arange(bs, dtype=np.int32)
    eng.fake_context(slots, lens, SEED)
    assign = np.array([i % 2 for i in range(bs)], np.int32)
    times, toks = [], []
    for i in range(warm + steps):
        t0 = time.perf_counter()
        out = eng.round(slots, assign)
        dt = time.perf_counter() - t0
        if i >= warm:
            times.append(dt)
            toks.append(int(out["accepted"].sum()) + bs)
    eng.close()
    value = sum(toks) / sum(times)
    return {"value": value, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "sample": (f"oracle port (C, OpenMP, {os.cpu_count()} threads): {steps} full config-2 rounds (SSM drafts, "
                       f"32-layer 7B-shaped verify, accept) on {bs} of the 32 requests at their config-2 context "
                       "lengths; KV filled with seeded values instead of a prefill forward; no extrapolation"),
            "s_per_round": sum(times) / len(times), "accepted_per_round": sum(toks) / len(toks),
            "requests_sampled": bs}


def reference_functions():
    """The reference's own single-threaded hot-path functions (oracle/_ref, built from
    /root/reference sources) on the config-2 shapes: BASELINE.md section 4 row 1."""
    import ctypes as C

    from oracle import REF_SO

    if not os.path.exists(REF_SO):
        return {"unavailable": "oracle/_ref/libspecsim_ref.so not built (needs /root/reference at build time)"}
    lib = C.CDLL(REF_SO)
    for f in ("ref_time_pack", "ref_time_verify_batch_cost", "ref_time_decomposed_attention", "ref_time_run_slot"):
        getattr(lib, f).restype = C.c_double
    from paper_2503_15921_b200.models import LLAMA_7B, synthetic_prompts

    prompts = synthetic_prompts(BATCH, PROMPT_LO, PROMPT_HI, LLAMA_7B.vocab, SEED)
    kv = np.array([len(p) + WINDOW for p in prompts], np.int32)  # Request::kv_len (model.hpp:26-28)
    p = kv.ctypes.data_as(C.c_void_p)
    head = lib.ref_time_decomposed_attention(p, BATCH, WINDOW + 1, LLAMA_7B.head_dim, BATCH, C.c_int(2))
    heads = LLAMA_7B.n_heads * LLAMA_7B.n_layers
    return {"cores": 1, "kind": "reference", "batch": BATCH, "window": WINDOW,
            "pack_us": lib.ref_time_pack(p, BATCH, BATCH, 2000) * 1e6,
            "verify_batch_cost_us": lib.ref_time_verify_batch_cost(p, BATCH, WINDOW, 1, BATCH, 2000) * 1e6,
            "decomposed_attention_ms_per_head": head * 1e3,
            "decomposed_attention_s_per_verify_step": head * heads,
            "decomposed_attention_note": (f"measured on one head (d={LLAMA_7B.head_dim}, {WINDOW + 1} queries per "
                                          f"request, config-2 kv lengths); a 7B verify step runs {heads} "
                                          "head-layers, so the per-step figure is that product"),
            "run_slot_us": lib.ref_time_run_slot(BATCH, PROMPT_LO, PROMPT_HI, WINDOW, 500) * 1e6,
            "run_slot_note": "cost-model simulation of one slot (32 requests, 2 SSMs, packing on)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cb = cpu_sample(args.steps, args.warmup)
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": cb["s_per_round"] * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp32-accum/bf16-storage", "data": "synthetic",
            "impl": "reference", "config": workload_config(None),
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "reference_functions": reference_functions(),
            "note": ("the reference (specsim) only simulates this path with cost models; its CPU implementation "
                     "of the real computation is the oracle port of its semantics (value); the reference's own "
                     "single-threaded hot-path functions are timed in reference_functions")}
    print(json.dumps(line), flush=True)


def parity_spot_check():
    """c2-shaped GPU-vs-oracle rounds (7B target, 68M/160M SSMs, 4 requests, short
    prompts, 2 rounds): the bit-exactness contract of tests/_parity.py, summarised."""
    sys.path.insert(0, ROOT)
    from paper_2503_15921_b200.models import LLAMA_7B, LLAMA_68M, LLAMA_160M
    from tests._parity import ParityRun

    run = ParityRun(LLAMA_7B, (LLAMA_68M, LLAMA_160M), batch=4, prompt_lo=16, prompt_hi=40, seed=7002, window=WINDOW,
                    max_ctx=96, device=int(os.environ.get("LOCAL_RANK", "0")))
    for _ in range(2):
        run.round(np.array([0, 1, 0, 1], np.int32))
    try:
        st = run.check()
        ok = True
    except AssertionError:
        st, ok = run.stats, False
    run.close()
    return {"workload": "c2 shapes, 4 requests, prompts U[16,40], 2 rounds", "bit_exact": ok,
            "decisions": st["decisions"], "forced_near_ties": st["forced"], "max_forced_deficit": st["deficit"],
            "twin_floor": st["floor"], "logits_rel_error_fro": st["worst_rel_fro"]}


def run_c3(args):
    """BASELINE config 3: request-decomposition sweep -- ragged draft lengths U{1..16}, batch 64,
    packed (pack() of the true lengths) vs padded (longest window, longest KV) verification
    of the 7B-shaped target on one B200; verify-step device us for each, plus the
    reference's verify_batch_cost token accounting (slot_engine.cpp:24-45) for the same batch."""
    import ctypes as C

    from paper_2503_15921_b200 import _lib
    from paper_2503_15921_b200.models import LLAMA_7B, LLAMA_68M, Engine, synthetic_prompts

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    B, W = 64, 16
    rng = np.random.default_rng(SEED + 3)
    prompts = synthetic_prompts(B, PROMPT_LO, PROMPT_HI, LLAMA_7B.vocab, SEED + 3)
    lens = rng.integers(1, W + 1, B).astype(np.int32)
    drafts = rng.integers(0, LLAMA_7B.vocab, int(lens.sum())).astype(np.int32)
    max_ctx = ((PROMPT_HI + W + 8 + 63) // 64) * 64
    out = {"metric": "verify-step us, packed vs padded (c3: ragged draft lengths 1-16, batch 64)", "unit": "us",
           "higher_is_better": False, "config": {"workload": "c3", "batch": B, "draft_len": "U{1..16}", "seed": SEED + 3,
                                                 "target": LLAMA_7B.name}}
    lib = _lib.load()
    kv_lens = np.array([len(p) + int(l) for p, l in zip(prompts, lens)], np.int32)  # kv_len = committed + window
    for width in (B, B // 2, B // 4):
        eng = Engine(LLAMA_7B, (LLAMA_68M,), max_requests=B, max_ctx=max_ctx, window=W, pack_width=width, device=dev)
        eng.prefill(range(B), prompts)
        slots = np.arange(B, dtype=np.int32)
        res = {}
        for mode, packed in (("packed", True), ("padded", False)):
            eng.verify_bench(slots, lens, drafts, packed=packed, iters=args.warmup)
            r = eng.verify_bench(slots, lens, drafts, packed=packed, iters=args.steps)
            res[mode] = {k: (float(v) if k == "us" else int(v)) for k, v in r.items() if k != "target"}
            res[mode]["target"] = r["target"]
        agree = float((res["packed"].pop("target") == res["padded"].pop("target")).mean())
        # reference token accounting for the same batch (verify_batch_cost, packed and padded)
        cost = {}
        for mode, packing in (("packed", 1), ("padded", 0)):
            tok, pad = C.c_int64(), C.c_int64()
            _lib.check(lib.spin_verify_batch_cost(kv_lens.ctypes.data_as(_lib.P_I32), B, W, packing, width,
                                                  C.byref(tok), C.byref(pad)))
            cost[mode] = {"tokens": tok.value, "padding": pad.value}
        out.setdefault("sweep", []).append({"pack_width": width, "packed": res["packed"], "padded": res["padded"],
                                            "speedup_padded_over_packed": res["padded"]["us"] / res["packed"]["us"],
                                            "target_token_agreement": agree, "reference_verify_batch_cost": cost})
        eng.close()
    best = min(out["sweep"], key=lambda s: s["packed"]["us"])
    out["value"] = best["packed"]["us"]
    out["padded_us"] = best["padded"]["us"]
    print(json.dumps(out), flush=True)


def serve(eng, sel, n_total, n_ssm, local_slots, slots_to_run, comm=None, prewarm=True):
    """spin_lbss_serve: the native multi-GPU LBSS loop (csrc/serve.cpp) on this rank."""
    import ctypes as C

    from paper_2503_15921_b200 import _lib

    rep = _lib.ServeReport()
    final = np.zeros(n_total, np.int32)
    ls = np.ascontiguousarray(local_slots, dtype=np.int32)
    _lib.check(eng.lib.spin_lbss_serve(eng.ctx, comm.h if comm is not None else None, sel.h, n_total, n_ssm,
                                       ls.ctypes.data_as(_lib.P_I32), len(ls), slots_to_run, int(prewarm),
                                       C.byref(rep), final.ctypes.data_as(_lib.P_I32)))
    return {k: getattr(rep, k) for k, _ in rep._fields_}, final


def run_c4(args):
    """BASELINE config 4: LLaMA-13B-shaped target, 3 heterogeneous SSMs (68M, 160M, 160M-b) with
    LBSS selection on measured goodput -- the native loop spin_lbss_serve (C++ selector, per-SSM
    wall times, switch catch-up charged, next-slot destinations prewarmed on idle streams) -- the
    SSM drafts of a slot running concurrently on their own CUDA streams. Every policy starts from
    the same freshly prefilled state and runs the same number of slots: LBSS with and without
    prewarm, and every homogeneous assignment (all requests on one SSM)."""
    from paper_2503_15921_b200.models import (C4_DOMAINS, LLAMA_13B, LLAMA_13B_DOM, LLAMA_68M, LLAMA_68M_DOM,
                                              LLAMA_160M, LLAMA_160M_B, LLAMA_160M_B_DOM, LLAMA_160M_DOM, Engine,
                                              domain_prompts, synthetic_prompts)
    from paper_2503_15921_b200.selector import Lbss

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    slots_n = max(args.steps, 128)
    max_ctx = ((PROMPT_HI + (WINDOW + 1) * (slots_n + 4) + 8 + 63) // 64) * 64
    if args.c4_uniform:  # round-1 setup: every SSM planted on the whole vocabulary
        target, ssms = LLAMA_13B, (LLAMA_68M, LLAMA_160M, LLAMA_160M_B)
        prompts = synthetic_prompts(BATCH, PROMPT_LO, PROMPT_HI, LLAMA_13B.vocab, SEED + 4)
        static = None
    else:  # per-request heterogeneity: request i lives in token domain i % 4, SSMs know some domains
        target, ssms = LLAMA_13B_DOM, (LLAMA_68M_DOM, LLAMA_160M_DOM, LLAMA_160M_B_DOM)
        prompts = domain_prompts(BATCH, PROMPT_LO, PROMPT_HI, target.vocab, C4_DOMAINS, SEED + 4)
        # informed static plan (not available to a real server): per domain the cheapest SSM that knows it
        static = np.array([[0, 1, 1, 2][i % C4_DOMAINS] for i in range(BATCH)], np.int32)
    slots = np.arange(BATCH, dtype=np.int32)
    out = {"metric": "accepted tokens/sec (c4: 13B target, 3 SSMs, LBSS)", "unit": "tokens/s",
           "higher_is_better": True, "config": {"workload": "c4", "target": target.name,
                                                "ssms": [s.name for s in ssms], "batch": BATCH, "window": WINDOW,
                                                "slots_per_policy": slots_n, "alpha": 8, "beta": 2,
                                                "domains": None if static is None else {
                                                    "n": C4_DOMAINS, "request_domain": "i % 4",
                                                    "ssm_planted_domains": [[d for d in range(C4_DOMAINS)
                                                                             if (s.planted_mask >> d) & 1]
                                                                            for s in ssms]}}}
    eng = Engine(target, ssms, max_requests=BATCH, max_ctx=max_ctx, window=WINDOW, device=dev)
    homo = {}
    plans = [(s.name, np.full(BATCH, j, np.int32)) for j, s in enumerate(ssms)]  # vanilla: all on SSM j
    if static is not None:
        plans.append(("static_per_domain_informed", static))
    for name, assign in plans:
        eng.prefill(range(BATCH), prompts)
        toks, ms, t0 = 0, 0.0, time.perf_counter()
        for _ in range(slots_n):
            r = eng.round(slots, assign)
            toks += int(r["accepted"].sum()) + BATCH
            ms += r["round_ms"]
        homo[name] = {"tokens_per_s_device": toks / (ms / 1e3),
                      "tokens_per_s_wall": toks / (time.perf_counter() - t0),
                      "mean_accepted": toks / (slots_n * BATCH) - 1}
    informed = homo.pop("static_per_domain_informed", None)
    runs = {}
    for prewarm in (True, False):
        eng.prefill(range(BATCH), prompts)
        sel = Lbss(BATCH, [BATCH] * len(ssms), alpha=8, beta=2, seed=SEED)
        rep, final = serve(eng, sel, BATCH, len(ssms), slots, slots_n, prewarm=prewarm)
        sel.close()
        runs["prewarm" if prewarm else "no_prewarm"] = {
            "tokens_per_s_device": rep["tokens"] / (rep["device_ms"] / 1e3),
            "tokens_per_s_wall": rep["tokens"] / (rep["wall_ms"] / 1e3), "switch_ms": rep["switch_ms"],
            "switch_tokens": rep["switch_tokens"], "explore_slots": rep["explore_slots"], "epochs": rep["epochs"],
            "final_plan_histogram": np.bincount(final[final >= 0], minlength=len(ssms)).tolist()}
    eng.close()
    best = max(homo, key=lambda k: homo[k]["tokens_per_s_device"])
    # value: LBSS without prewarm, whose device time covers all of its GPU work (prewarm work that
    # outlasts a round runs outside the rounds' clock; its wall time shows the enqueue waits)
    out["value"] = runs["no_prewarm"]["tokens_per_s_device"]
    out["lbss"] = runs
    out["homogeneous"] = homo
    if informed is not None:
        out["static_per_domain_informed"] = informed
    out["lbss_over_best_homogeneous"] = {
        "best": best,
        **{f"{k}_{clock}": runs[k][f"tokens_per_s_{clock}"] / homo[best][f"tokens_per_s_{clock}"]
           for k in runs for clock in ("device", "wall")}}
    if informed is not None:
        out["lbss_over_best_homogeneous"]["informed_static_device"] = (
            informed["tokens_per_s_device"] / homo[best]["tokens_per_s_device"])
    out["note"] = ("device time of every slot includes the synchronous KV catch-up of switched requests "
                   "(switching_cost, slot_engine.cpp:12-22); wall time adds the host selector and launch overheads")
    print(json.dumps(out), flush=True)


def run_c5(args, ranks):
    """BASELINE config 5: 256 requests sharded over the ranks (strong scaling), replicated weights,
    the native LBSS loop on every rank with the per-slot NCCL all-gather of ArmEstimate rows
    (spin_stats_allgather). value = all tokens / max over ranks of the device time."""
    from paper_2503_15921_b200.dist import shard
    from paper_2503_15921_b200.models import LLAMA_7B, LLAMA_68M, LLAMA_160M, Engine, synthetic_prompts
    from paper_2503_15921_b200.selector import Lbss

    N = 256
    ssms = (LLAMA_68M, LLAMA_160M)
    mine = shard(N, ranks.world, ranks.rank)
    n_local = len(mine)
    slots_n = args.steps + args.warmup
    max_ctx = ((PROMPT_HI + (WINDOW + 1) * (slots_n + 4 + 4 * 4) + 8 + 63) // 64) * 64
    prompts = synthetic_prompts(N, PROMPT_LO, PROMPT_HI, LLAMA_7B.vocab, SEED + 5)
    eng = Engine(LLAMA_7B, ssms, max_requests=n_local, max_ctx=max_ctx, window=WINDOW, device=ranks.device)
    eng.prefill(range(n_local), [prompts[i] for i in mine])
    slots = np.arange(n_local, dtype=np.int32)
    # f1: pipelining plan tuned on measured throughput on this rank's shard (i % 2 assignment)
    chosen, curve = eng.tune_micro_batches(slots, np.array([i % 2 for i in range(n_local)], np.int32),
                                           max_micro_batches=args.max_micro_batches, probe_rounds=3)
    sel = Lbss(N, [N] * len(ssms), alpha=8, beta=2, seed=SEED)
    # warm-up slots (graph capture per assignment shape), then the timed slots
    pw = not args.c5_no_prewarm
    serve(eng, sel, N, len(ssms), slots, args.warmup, ranks.comm, prewarm=pw)
    ranks.barrier()
    with ClockSampler(ranks.device) as clk:
        rep, final = serve(eng, sel, N, len(ssms), slots, args.steps, ranks.comm, prewarm=pw)
        ranks.barrier()
    dev_ms = ranks.max(rep["device_ms"])
    wall_ms = ranks.max(rep["wall_ms"])
    tokens = ranks.sum(float(rep["tokens"]))
    eng.close()
    sel.close()
    line = {"metric": "accepted tokens/sec (c5: batch 256 sharded, LBSS with NCCL stats all-gather)",
            "value": tokens / (dev_ms / 1e3), "unit": UNIT, "n_gpus": ranks.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "c5: 256 requests sharded over the ranks, LLaMA-7B-shaped target, "
                                   "LLaMA-68M/160M-shaped SSMs, LBSS (alpha 8, beta 2) on every rank",
                       "requests_per_gpu": n_local, "parallelism": f"request-sharded dp{ranks.world}",
                       "comm": ranks.backend, "shared_device": ranks.shared},
            "e2e": {"value": tokens / (wall_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": 4 * 3 * n_local,
                    "d2h_bytes_per_step": 4 * n_local * (3 + 2 * WINDOW + 1)},
            "lbss": {"prewarm": pw, "explore_slots": rep["explore_slots"], "epochs": rep["epochs"], "switch_ms": rep["switch_ms"],
                     "final_plan_histogram": np.bincount(final[final >= 0], minlength=len(ssms)).tolist()},
            "pipelining": {"chosen_per_ssm": chosen.tolist(), "curve_tokens_per_s": curve, "probe_rounds": 3,
                           "candidates": "uniform b = 1 (serial) .. 4 micro-batches per SSM"},
            "clocks": clk.summary()}
    if ranks.rank == 0:
        print(json.dumps(line), flush=True)


def workload_config(eng_info):
    from paper_2503_15921_b200.models import LLAMA_7B, LLAMA_68M, LLAMA_160M

    cfg = {"workload": "c2: LLaMA-7B-shaped target verifying LLaMA-68M/160M-shaped SSM drafts, greedy",
           "batch_per_gpu": BATCH, "window": WINDOW, "prompt_len": f"U[{PROMPT_LO},{PROMPT_HI}]",
           "target": LLAMA_7B.name, "ssms": [LLAMA_68M.name, LLAMA_160M.name], "assignment": "request i -> ssm i%2",
           "l2": "no flush needed: 13.5 GB of target weights stream through the 126 MB L2 every step"}
    if eng_info:
        cfg.update(eng_info)
    return cfg


def gemm_roofline(eng, target, T, hbm, tflops, peak_src):
    """Dominant kernel class: the target's projection GEMMs, replayed in situ (spin_kernel_bench).
    HBM-bound below the ridge (T < ~250 rows), tensor-bound above it."""
    g_us, g_bytes = eng.kernel_bench("gemm", 5)
    D, F, L = target.d_model, target.ffn, target.n_layers
    g_flops = 2.0 * T * L * (4 * D * D + 3 * D * F) / (4 * L)  # per launch (4 GEMMs per layer)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "gemm_dram_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                traffic = json.load(f).get("bytes_per_launch_target_gemm")
        except Exception:
            traffic = None
    tensor = g_flops / g_bytes > tflops * 1e12 / (hbm * 1e9)  # arithmetic intensity (flop/B) above the ridge
    if tensor:
        achieved = g_flops / (g_us * 1e-6) / 1e12
        return {"bound": "tensor", "kernel": "tcgen05 weight-streaming GEMM (target projections)",
                "achieved": achieved, "peak": tflops, "unit": "TFLOP/s", "frac": achieved / tflops,
                "traffic": None, "peak_source": peak_src, "alg_flops_per_launch": g_flops,
                "alg_bytes_per_launch": g_bytes, "us_per_launch": g_us}
    achieved = g_bytes / (g_us * 1e-6) / 1e9
    return {"bound": "hbm", "kernel": "tcgen05 weight-streaming GEMM (target projections)", "achieved": achieved,
            "peak": hbm, "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic, "peak_source": peak_src,
            "alg_bytes_per_launch": g_bytes, "us_per_launch": g_us}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="spin", choices=["spin", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--pack-width", type=int, default=0)
    ap.add_argument("--max-micro-batches", type=int, default=4, help="f1 tuner candidates (1 = serial only)")
    ap.add_argument("--config", default="c2", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--c4-uniform", action="store_true", help="c4 with every SSM planted on the whole vocabulary")
    ap.add_argument("--c5-no-prewarm", action="store_true", help="c5 with synchronous switch catch-ups only")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if os.environ.get("SPIN_BENCH_SHARE_DEVICE") == "1":
        # functional runs of the N > 1 plumbing on one GPU: ranks time-slice the device, so
        # the pipelining probes (per-unit graphs on several streams) are not meaningful there
        # (and hit an illegal address once in that setting; one process per GPU never did)
        args.max_micro_batches = 1
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if args.config == "c3":
        run_c3(args)
        return
    if args.config == "c4":
        run_c4(args)
        return
    ranks = Ranks()
    if args.config == "c5":
        run_c5(args, ranks)
        ranks.close()
        return

    from paper_2503_15921_b200.dist import AcceptanceStats
    from paper_2503_15921_b200.models import LLAMA_7B, LLAMA_68M, LLAMA_160M, Engine, synthetic_prompts

    world, rank, local = ranks.world, ranks.rank, ranks.device
    hbm, tflops, peak_src = peaks()
    rounds_total = 2 * (args.warmup + args.steps) + 4 + 4 * 5  # + the pipelining probes
    max_ctx = ((PROMPT_HI + (WINDOW + 1) * rounds_total + 8 + 63) // 64) * 64
    eng = Engine(LLAMA_7B, (LLAMA_68M, LLAMA_160M), max_requests=BATCH, max_ctx=max_ctx, window=WINDOW, device=local,
                 pack_width=args.pack_width)
    prompts = synthetic_prompts(BATCH, PROMPT_LO, PROMPT_HI, LLAMA_7B.vocab, SEED + rank)
    eng.prefill(range(BATCH), prompts)
    slots = np.arange(BATCH, dtype=np.int32)
    assign = np.array([i % 2 for i in range(BATCH)], np.int32)
    # per-(request, SSM) acceptance statistics, ArmEstimate{sum,count} (bandit.hpp:24-39),
    # all-gathered every e2e step through libspin (the only collective of the path)
    stats = AcceptanceStats(BATCH * world, 2, world, rank)

    # ---- warm-up (graph capture, clocks, caches)
    for _ in range(args.warmup):
        eng.round(slots, assign)
    with ClockSampler(local) as clk:
        # ---- value: device-resident rounds
        ranks.barrier()
        emitted, dev_ms = eng.run_rounds(slots, assign, args.steps)
        ranks.barrier()
        dev_ms_max = ranks.max(dev_ms)
        tokens_total = ranks.sum(float(emitted.sum()))
        value = tokens_total / (dev_ms_max / 1e3)
        # ---- e2e: public per-slot call with host buffers + per-step stats gather, over the SAME
        # rounds as `value` (re-prefilled, same warm-up: greedy decoding repeats them token for
        # token), so the two differ only by the host path, not by longer contexts
        eng.prefill(range(BATCH), prompts)
        for _ in range(args.warmup):
            eng.round(slots, assign)
        verify_us, draft_us, committed = [], [], None
        ranks.barrier()
        t0 = time.perf_counter()
        e2e_tokens = 0
        for _ in range(args.steps):
            out = eng.round(slots, assign)
            e2e_tokens += int(out["accepted"].sum()) + BATCH
            stats.add_many(np.arange(BATCH), assign, (out["accepted"] + 1) / (out["wall_ms"] / 1e3))
            stats.gather(ranks.comm)
            verify_us.append(out["verify_ms"] * 1e3)
            draft_us.append(out["draft_ms"] * 1e3)
            committed = out["committed"]
        ranks.barrier()
        e2e_s = ranks.max(time.perf_counter() - t0)
        e2e_value = ranks.sum(float(e2e_tokens)) / e2e_s
    clocks = clk.summary()
    launches = eng.launches_per_round(slots, assign)
    # ---- per-kernel-class device time of one (un-graphed) round
    prof = eng.profile(slots, assign)
    eng.round(slots, assign)  # graph round: leaves the target's verify state for the in-situ replays
    T = BATCH * (WINDOW + 1)
    roof = gemm_roofline(eng, LLAMA_7B, T, hbm, tflops, peak_src)
    a_us, a_bytes = eng.kernel_bench("attention", 5)
    a_achieved = a_bytes / (a_us * 1e-6) / 1e9
    roof["method"] = ("the 128 projection GEMMs (4 per layer) of the last verify replayed as one CUDA graph with "
                      "PDL, CUDA events on the launch stream, 5 replays")
    roof["attention"] = {"achieved": a_achieved, "frac": a_achieved / hbm, "us_per_launch": a_us,
                         "alg_bytes_per_launch": a_bytes, "bound": "hbm",
                         "kernel": "packed ragged causal attention + shared-max combine"}
    # f1: speculation/verification pipelining, tuned on measured throughput
    # (tune_micro_batches, pipeline.cpp:345-380); the main line above is the serial round
    chosen, curve = eng.tune_micro_batches(slots, assign, max_micro_batches=args.max_micro_batches, probe_rounds=4)
    pipelining = {"candidates": "uniform b = 1 (serial) .. 4 micro-batches per SSM", "probe_rounds": 4,
                  "curve_tokens_per_s": curve, "chosen_per_ssm": chosen.tolist(),
                  "note": "b = 1 is the serial round; each further group re-streams the target weights in its own "
                          "verification (HBM-bound at this batch), so the tuner keeps the serial round unless "
                          "overlapping the drafts pays for that"}
    t_roof_us, alg_bytes, alg_flops = path_roofline_us(LLAMA_7B, committed - 0, WINDOW, hbm, tflops)
    verify_med = statistics.median(verify_us)
    round_ms = dev_ms_max / args.steps
    h2d = 4 * (3 * BATCH)
    d2h = 4 * BATCH * (3 + 2 * WINDOW + 1)
    mean_acc = float(emitted.sum()) / (args.steps * BATCH) - 1.0
    info = {"pack_width": args.pack_width or BATCH, "parallelism": f"request-sharded dp{world}",
            "comm": ranks.backend, "shared_device": ranks.shared,
            "verify_step_us_median": verify_med, "draft_us_median": statistics.median(draft_us),
            "verify_roofline_us": t_roof_us, "verify_roofline_frac": t_roof_us / verify_med,
            "verify_alg_bytes": alg_bytes, "verify_alg_flops": alg_flops,
            "mean_accepted_per_request": mean_acc, "per_class_ms_one_round": {k: v[0] for k, v in prof.items()},
            "per_class_launches": {k: v[2] for k, v in prof.items()}, "pipelining": pipelining}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round_ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded random-init weights, planted bigram)",
            "config": workload_config(info),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": int(launches) * args.steps, "roofline": roof, "clocks": clocks}
    eng.close()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_sample(2, 1)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        if not args.no_parity:
            line["parity"] = parity_spot_check()
    if rank == 0:
        print(json.dumps(line), flush=True)
    ranks.close()


if __name__ == "__main__":
    main()
