/*
 * spin_c.h -- the C-ABI drop-in boundary of the B200 Spin verification path.
 *
 * Plain C types only (pointers, sizes, PODs); no C++ or torch types. Every entry
 * point returns a spin_status; spin_last_error() holds a thread-local message.
 * The C++ host layer (include/specsim/ headers) rethrows each status as the
 * reference's exception type, so reference callers stay unchanged.
 *
 * Reference interfaces replaced (paths under /root/reference/proj/core):
 *   status codes        <- include/specsim/errors.hpp:7-33 (ConfigError .. IoError) + CUDA
 *   spin_pack           <- include/specsim/packing.hpp:52  pack(kv_lens, width)
 *   spin_naive_padding  <- include/specsim/packing.hpp:56  naive_padding(kv_lens)
 *   spin_verify_batch_cost <- include/specsim/slot_engine.hpp:98-99 verify_batch_cost(...)
 *   spin_decomposed_attention <- include/specsim/attention.hpp:42-44 decomposed_attention(...)
 *   spin_reference_attention  <- include/specsim/attention.hpp:34 reference_attention(q,k,v)
 *   spin_ctx_* / spin_prefill / spin_round <- include/specsim/slot_engine.hpp:50-88
 *        SlotEngine ctor + run_slot (speculate -> verify -> accept -> update),
 *        with the Bernoulli draw of src/model.cpp:110-134 replaced by real greedy
 *        verification of SSM drafts against the target model.
 */
#ifndef SPIN_C_H_
#define SPIN_C_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPIN_ABI_VERSION 3
#define SPIN_MAX_SSM 8

typedef enum spin_status {
  SPIN_OK = 0,
  SPIN_CONFIG_ERROR = 1,      /* specsim::ConfigError      */
  SPIN_CAPACITY_ERROR = 2,    /* specsim::CapacityError    */
  SPIN_INPUT_ERROR = 3,       /* specsim::InputError       */
  SPIN_SIZE_ERROR = 4,        /* specsim::SizeError        */
  SPIN_CONSISTENCY_ERROR = 5, /* specsim::ConsistencyError */
  SPIN_METRIC_ERROR = 6,      /* specsim::MetricError      */
  SPIN_IO_ERROR = 7,          /* specsim::IoError          */
  SPIN_CUDA_ERROR = 8         /* device / driver failure (no reference equivalent) */
} spin_status;

int spin_abi_version(void);
const char* spin_last_error(void);

/* ------------------------------------------------------------------------
 * Request decomposition (packing.hpp:10-59, packing.cpp:16-136). Host-side,
 * bit-identical to the reference's first-fit-decreasing packer.
 * ---------------------------------------------------------------------- */
typedef struct spin_segment {
  int32_t request_id;
  int32_t row;
  int32_t col_start;
  int32_t col_end; /* exclusive */
  int32_t token_offset;
} spin_segment;

/* segments must hold seg_cap >= n + min(width, n) - 1 entries (the packer's
 * bound); q_replica_rows holds n entries. Empty input -> length = rows = 0. */
spin_status spin_pack(const int32_t* kv_lens, int32_t n, int32_t width, int32_t* length, int32_t* rows,
                      spin_segment* segments, int32_t seg_cap, int32_t* n_segments, int64_t* padding_tokens,
                      int32_t* q_replica_rows);
spin_status spin_naive_padding(const int32_t* kv_lens, int32_t n, int64_t* padding);
spin_status spin_verify_batch_cost(const int32_t* kv_lens, int32_t n, int32_t window, int32_t packing,
                                   int32_t pack_width, int64_t* tokens, int64_t* padding);

/* Device request decomposition: the packer the hot path runs (meta_kernel, one warp:
 * ballot first-fit + warp-scan splits), launched on its own. Same contract and error
 * taxonomy as spin_pack; bit-identical to it (tests/test_gpu_pack_device.py pins it to
 * the reference goldens). n <= 1024. */
spin_status spin_pack_device(const int32_t* kv_lens, int32_t n, int32_t width, int32_t* length, int32_t* rows,
                             spin_segment* segments, int32_t seg_cap, int32_t* n_segments,
                             int64_t* padding_tokens, int32_t* q_replica_rows);

/* ------------------------------------------------------------------------
 * Packed (decomposed) attention operator in the reference's toy mode
 * (attention.cpp:67-162: fp64, scale 1, no causal mask, any dim). Host buffers
 * in fp64 like the reference Matrix; computed on the device in fp64 by a
 * dedicated split-KV kernel (launch_toy_attention in kernels.cu) -- one partial
 * per (segment, query) and the shared-max combine across a request's segments.
 * It is NOT the production verifier kernel (bf16 KV, head_dim 64/128, causal);
 * spin_attention below runs that one. q/k/v are the per-request matrices
 * concatenated row-major: q rows sum(q_rows[i]), k/v rows sum(kv_rows[i]).
 * mask (width*length owner ids, -1 empty) is checked against the layout like
 * check_layout_consistency (attention.cpp:23-63); pass NULL to skip.
 * ---------------------------------------------------------------------- */
spin_status spin_decomposed_attention(int32_t n_req, int32_t dim, const int32_t* q_rows, const int32_t* kv_rows,
                                      const double* q, const double* k, const double* v, const spin_segment* segs,
                                      int32_t n_segs, int32_t width, int32_t length, const int32_t* mask,
                                      double* out);
spin_status spin_reference_attention(int32_t q_rows, int32_t kv_rows, int32_t dim, const double* q,
                                     const double* k, const double* v, double* out);

/* ------------------------------------------------------------------------
 * Verification engine (one context per GPU / process).
 * ---------------------------------------------------------------------- */
typedef struct spin_model_desc {
  int32_t d_model;
  int32_t n_layers;
  int32_t n_heads;
  int32_t head_dim; /* 64 or 128 */
  int32_t ffn;
  int32_t vocab;
  float rope_theta;
  float rms_eps;
  uint64_t seed;     /* synthetic weight stream */
  float embed_scale; /* embedding entries ~ U(-a, a) * embed_scale          */
  float planted_gain;/* strength of the planted next-token map in lm_head    */
  float resid_scale; /* o_proj / down_proj scale: block contribution size    */
  float init_scale;  /* other projections ~ U(-1,1) * init_scale             */
  /* Token domains of the planted map (ABI v3): the vocabulary splits into planted_domains
   * contiguous ranges of vocab / planted_domains ids and pi maps every range onto itself;
   * the lm_head rows of domain d carry the planted term only if bit d of planted_mask is
   * set. 0 / 0 = one domain, all planted (the v2 behaviour). A model whose mask misses a
   * request's domain drafts noise for it: per-request heterogeneous SSM quality (config 4). */
  int32_t planted_domains;
  uint32_t planted_mask;
} spin_model_desc;

typedef struct spin_engine_opts {
  int32_t device;
  int32_t max_requests; /* request slots (KV cache rows) */
  int32_t max_ctx;      /* positions per slot            */
  int32_t window;       /* gamma                         */
  int32_t pack_width;   /* 0: batch size (slot_engine.cpp:30-31)            */
  int32_t packing;      /* 1: decomposed split-KV work list, 0: padded rows */
  int32_t use_graphs;   /* capture draft/verify in CUDA graphs              */
  int32_t use_pdl;      /* programmatic dependent launch between kernels    */
  int32_t debug_logits; /* keep fp32 target logits of the last verify       */
} spin_engine_opts;

typedef struct spin_ctx spin_ctx;

spin_status spin_ctx_create(const spin_model_desc* target, const spin_model_desc* ssms, int32_t n_ssm,
                            const spin_engine_opts* opts, spin_ctx** out);
spin_status spin_ctx_destroy(spin_ctx* ctx);

/* Admits n requests into the given slots and runs the prompt prefill on the
 * target and every SSM. prompts: concatenated token ids, prompt_lens[i] >= 2.
 * The last prompt token stays pending (it is the first verify row). */
spin_status spin_prefill(spin_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* prompt_lens,
                         const int32_t* prompts);

typedef struct spin_round_out {
  int32_t* accepted;      /* [n] leading-run length, 0..window          */
  int32_t* bonus_token;   /* [n] target token after the accepted run    */
  int32_t* committed;     /* [n] committed tokens after the round       */
  int32_t* drafts;        /* [n*window] or NULL                         */
  int32_t* target_tokens; /* [n*(window+1)] target argmax rows or NULL  */
  float draft_ms;         /* device time: all SSM draft loops           */
  float verify_ms;        /* device time: pack + verify forward + accept */
  float round_ms;         /* device time: whole round, switch catch-up included */
  float switch_ms;        /* device time of the synchronous KV catch-up of requests whose SSM
                             cache lags (switches, switching_cost slot_engine.cpp:12-22); 0 if none */
  int32_t switch_tokens;  /* KV positions recomputed by that catch-up */
  float spec_end_ms[SPIN_MAX_SSM]; /* per SSM: draft end, ms after the draft start (-1: idle); the
                             request's wall time is spec_end_ms[ssm] + verify_ms (slot_engine.cpp:145) */
  int32_t* switch_tokens_per_request; /* [n] or NULL: positions recomputed per request */
} spin_round_out;

/* One speculation + verification slot for n admitted requests. ssm_of[i] is
 * the draft model of request i (slots[i]); -1 idles it (not verified). Host
 * buffers; H2D of the assignment and D2H of the outcome are inside the call. */
spin_status spin_round(spin_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* ssm_of,
                       spin_round_out* out);
/* spin_round plus prewarm (run_slot's `prewarm`, slot_engine.hpp:50-88): prewarm[i]
 * (or -1) names the SSM request i is expected to move to; its KV is recomputed up
 * to the committed prefix on that SSM's idle stream WHILE this round runs
 * (prewarm_destination, bandit.cpp:122-139), so the later switch only catches up
 * the last round's commits. Later calls order themselves after it on the device. */
spin_status spin_round_prewarm(spin_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* ssm_of,
                               const int32_t* prewarm, spin_round_out* out);

/* Device-resident loop: one host-driven spin_round first (validation, SSM
 * switches, graph capture; its outcome is not reported), then `rounds` rounds
 * back to back on the current assignment with no host round trip -- rounds + 1
 * rounds in total, so every active slot needs committed + (rounds + 1) * (window + 1)
 * <= max_ctx (else SPIN_CAPACITY_ERROR, nothing runs). Per-round accepted+bonus
 * totals of the `rounds` timed rounds land in emitted[rounds] (host) after the
 * final synchronisation. */
spin_status spin_run_rounds(spin_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* ssm_of,
                            int32_t rounds, int64_t* emitted, float* device_ms);

/* Speculation/verification pipelining (pipeline.cpp:160-329): per SSM, its
 * requests are split into per_ssm[j] micro-batch groups (near-equal, batch order);
 * with any count above 1, each (SSM, group) drafts on the SSM's stream and is
 * verified on its own, FIFO in expected arrival order, and in spin_run_rounds the
 * next slot's draft of a group starts as soon as that group was verified
 * (causality, pipeline.cpp:236-241) -- drafting overlaps verification. All ones
 * (the default) is the serial round: every SSM drafts, one packed verification.
 * Outcomes follow the same greedy semantics either way. */
spin_status spin_set_micro_batches(spin_ctx* ctx, const int32_t* per_ssm, int32_t n_ssm);
spin_status spin_get_micro_batches(spin_ctx* ctx, int32_t* per_ssm, int32_t n_ssm);
/* tune_micro_batches (pipeline.cpp:345-380) on MEASURED throughput: uniform plans
 * b = 1, 2 .. max_micro_batches (capped by the largest SSM batch), each probed with
 * probe_rounds device-resident rounds (spin_run_rounds) on the given requests; stops
 * at the first plan more than `threshold` below the best and keeps the last
 * non-degraded one (set on the context, copied to chosen[n_ssm]); curve[k] = the
 * measured accepted tokens/s of candidate k. The probes commit tokens (real rounds). */
spin_status spin_tune_micro_batches(spin_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* ssm_of,
                                    int32_t max_micro_batches, int32_t probe_rounds, double threshold,
                                    int32_t* chosen, double* curve, int32_t curve_cap, int32_t* n_curve);

/* Committed token history of one slot (prompt + generated). */
spin_status spin_read_tokens(spin_ctx* ctx, int32_t slot, int32_t* tokens, int32_t cap, int32_t* len);
/* fp32 target logits of the last verify ([rows, vocab]); needs debug_logits. */
spin_status spin_read_logits(spin_ctx* ctx, float* logits, int64_t cap, int32_t* rows);
/* Rebinds a request slot to a different SSM: the SSM's KV for the slot is
 * recomputed up to the committed prefix (switching_cost, slot_engine.cpp:12-22). */
spin_status spin_switch_ssm(spin_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* ssm_of);

/* Profiling: one round run without graphs, CUDA events around every launch.
 * Arrays have SPIN_PROF_CLASSES entries indexed by class: device ms, algorithmic
 * bytes (GEMM classes: weights + activations in + out), and launch counts. */
#define SPIN_PROF_CLASSES 9
enum {
  SPIN_PROF_TARGET_GEMM = 0,
  SPIN_PROF_TARGET_HEAD = 1,
  SPIN_PROF_TARGET_ATTN = 2,
  SPIN_PROF_TARGET_EPI = 3,
  SPIN_PROF_SSM_GEMM = 4,
  SPIN_PROF_SSM_HEAD = 5,
  SPIN_PROF_SSM_ATTN = 6,
  SPIN_PROF_SSM_EPI = 7,
  SPIN_PROF_META = 8
};
spin_status spin_profile_round(spin_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* ssm_of, double* ms,
                               double* bytes, int64_t* launches);
/* Kernels launched per round for this assignment shape (after a first round). */
spin_status spin_round_launches(spin_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* ssm_of,
                                int64_t* launches);

/* In-situ kernel timing on the target state of the last verify: kind 0 = the
 * four projection GEMMs of every layer, kind 1 = attention (split-KV merge in-kernel) of every
 * layer, replayed as one CUDA graph `iters` times (CUDA events). Outputs the
 * average device time per launch and algorithmic bytes per launch. */
spin_status spin_kernel_bench(spin_ctx* ctx, int32_t kind, int32_t iters, double* us_per_launch,
                              double* bytes_per_launch);

/* Event trace of the last spin_round: per-SSM draft end, device ms after the
 * round start (-1 for an SSM without requests). With draft_ms (= verify start),
 * round_ms (= verify end) of spin_round_out this yields the reference's
 * EventTrace (pipeline.hpp:14-30): spec_start/spec_end per SSM, verify_start/end. */
spin_status spin_last_round_trace(spin_ctx* ctx, float* spec_end_ms, int32_t cap);

/* Ragged-window verification (BASELINE config 3, request-decomposition sweep):
 * request i verifies draft_lens[i] in 1..window drafts (drafts: host tokens, flat,
 * sum(draft_lens) entries, or NULL for the history token). packed = 1: pack() of
 * the true lengths (sum(len+1) query rows); 0: padded to the longest window and
 * the longest KV (the reference's naive_padding baseline, slot_engine.cpp:37-44).
 * Nothing is committed; `iters` graph replays are timed with CUDA events. */
typedef struct spin_verify_stats {
  double us;               /* device microseconds per verification step */
  int64_t query_rows;      /* rows through the target forward (incl. padding) */
  int64_t real_rows;       /* sum(draft_lens + 1) */
  int64_t kv_tokens;       /* KV tokens the attention reads (incl. padding) */
  int32_t* target_tokens;  /* optional host [sum(draft_lens + 1)]: target argmax of each real row */
} spin_verify_stats;
spin_status spin_verify_bench(spin_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* draft_lens,
                              const int32_t* drafts, int32_t packed, int32_t iters, spin_verify_stats* out);

/* ------------------------------------------------------------------------
 * Multi-GPU exchange: requests shard across ranks
 * (one process per GPU, replicated weights); the only collective of the path is
 * an all-gather of the selector's per-(request, SSM) ArmEstimate{sum, count}
 * rows (bandit.hpp:24-39; update sites bandit.cpp:166-169, policies.cpp:69-72).
 * A communicator spans processes, so it is its own handle (one per device)
 * rather than part of spin_ctx. Backends: NCCL (ncclAllGather over NVLink,
 * libnccl loaded at first use) and TCP (same semantics, no GPU: CPU tests).
 * id: NCCL -> the ncclUniqueId bytes from rank 0's spin_comm_unique_id, shared
 * out of band; TCP -> "ipv4:port" of rank 0 (spin_comm_unique_id picks a free
 * loopback port). Results are rank-ordered and identical on every rank.
 * ---------------------------------------------------------------------- */
#define SPIN_COMM_ID_BYTES 128
enum { SPIN_COMM_NCCL = 0, SPIN_COMM_TCP = 1 };
enum { SPIN_REDUCE_SUM = 0, SPIN_REDUCE_MAX = 1 };
typedef struct spin_comm spin_comm;
spin_status spin_comm_unique_id(int32_t backend, uint8_t* id /* SPIN_COMM_ID_BYTES */);
spin_status spin_comm_create(int32_t backend, int32_t device, int32_t rank, int32_t world, const uint8_t* id,
                             spin_comm** out);
spin_status spin_comm_destroy(spin_comm* comm);
spin_status spin_comm_info(spin_comm* comm, int32_t* rank, int32_t* world, int32_t* backend);
/* local: this rank's rows [rows][m][2] = {sum, count} (every rank passes the same
 * `rows`: pad the shards to the largest); global: [world * rows][m][2], rank-major. */
spin_status spin_stats_allgather(spin_comm* comm, const double* local, double* global, int32_t rows, int32_t m);
/* In-place element-wise reduction over ranks (rank order, deterministic). */
spin_status spin_comm_allreduce(spin_comm* comm, double* values, int32_t n, int32_t op);
spin_status spin_comm_barrier(spin_comm* comm);

/* ------------------------------------------------------------------------
 * LBSS, the learning-based SSM selector (host side; bandit.cpp:11-332 restated in
 * C++: same Rng draw order, schedule and tie-breaking as the reference, pinned by
 * tests/test_lbss.py to traces of the reference's own functions). Every request is
 * admitted. next() yields the slot's assignment [n] (ssm or -1), the prewarm
 * destinations [n] (exploration: the chunk's draw; exploitation: the optimistic
 * argmax decided before the matching), the explore flag and the epoch. observe()
 * is ArmEstimate::add(observed_goodput) (bandit.cpp:166-169). rows() reads (set=0)
 * or replaces (set=1) all estimates as [n][m][2] = {sum, count}: the multi-GPU
 * driver replaces them with the all-gathered rows every slot.
 * ---------------------------------------------------------------------- */
typedef struct spin_lbss spin_lbss;
spin_status spin_lbss_create(int32_t n_requests, int32_t n_ssm, const int32_t* capacities, int32_t alpha,
                             int32_t beta, uint64_t seed, spin_lbss** out);
spin_status spin_lbss_destroy(spin_lbss* sel);
spin_status spin_lbss_next(spin_lbss* sel, int32_t* assignment, int32_t* prewarm, int32_t* explore, int32_t* epoch);
spin_status spin_lbss_observe(spin_lbss* sel, int32_t request, int32_t ssm, double goodput);
spin_status spin_lbss_rows(spin_lbss* sel, double* rows, int32_t set);
/* plan_exploitation on the current estimates (no schedule state change). */
spin_status spin_lbss_plan(spin_lbss* sel, int32_t* assignment);
/* The next slot's assignment where already determined (prewarm planning): the
 * current one inside a chunk / stage, the next chunk's draw at a chunk boundary
 * (same Rng sequence), prewarm_destination before the first exploitation slot. */
spin_status spin_lbss_peek(spin_lbss* sel, int32_t* assignment);

/* The multi-GPU serving loop (csrc/serve.cpp): `slots_to_run` LBSS slots over
 * this rank's contiguous shard (local_slots, n_local = the shard size of n_total
 * requests over the communicator's ranks; comm may be NULL for one rank): per slot
 * the selector's assignment, spin_round_prewarm (next slot's destinations warmed),
 * observed goodput into the local ArmEstimate rows, spin_stats_allgather, and the
 * gathered rows replacing the selector's estimates on every rank. */
typedef struct spin_serve_report {
  double device_ms;       /* sum of round_ms (switch catch-up included), this rank */
  double wall_ms;         /* host wall time of the loop, this rank (gathers included) */
  int64_t tokens;         /* accepted + bonus, this rank */
  int64_t served;         /* request-slots served, this rank */
  int32_t explore_slots;
  int32_t epochs;
  double switch_ms;       /* synchronous switch catch-up inside device_ms */
  int64_t switch_tokens;  /* KV positions recomputed synchronously */
} spin_serve_report;
spin_status spin_lbss_serve(spin_ctx* ctx, spin_comm* comm, spin_lbss* sel, int32_t n_total, int32_t n_ssm,
                            const int32_t* local_slots, int32_t n_local, int32_t slots_to_run, int32_t use_prewarm,
                            spin_serve_report* rep, int32_t* final_assignment /* [n_total]: the plan on the
                                                                                final estimates, or NULL */);

/* ------------------------------------------------------------------------
 * Device plumbing: lets callers (and the parity tests) hold device buffers
 * without any framework. spin_device_count reports 0 (status OK) when there is
 * no driver or device. spin_device_alloc zero-fills. kind: 1 H2D, 2 D2H, 3 D2D.
 * ---------------------------------------------------------------------- */
spin_status spin_device_count(int32_t* count);
spin_status spin_device_alloc(int32_t device, size_t bytes, void** ptr);
spin_status spin_device_free(void* ptr);
spin_status spin_memcpy(void* dst, const void* src, size_t bytes, int32_t kind);

/* ------------------------------------------------------------------------
 * Kernel-level entry points (device pointers; stream = cudaStream_t or NULL).
 * Used by the parity tests to check each kernel against a reference of the
 * same op, and by bench.py for the per-kernel roofline.
 * ---------------------------------------------------------------------- */
spin_status spin_gemm_info(int32_t n_out, int32_t k, int32_t t, int32_t mode, int32_t* max_pieces,
                           int32_t* grid, int32_t* bn);
/* w: row-major [n_out][k] bf16 (converted to the tiled GEMM weight layout internally); x: [t][k].
 * mode 0: part[max_pieces][t][n_out] partial sums (caller zero-fills, sums slots);
 * mode 1: amax_val/amax_idx [ceil(n_out/128)][t], logits [t][n_out] optional. Synchronous. */
spin_status spin_gemm(void* stream, const void* w, const void* x, int32_t n_out, int32_t k, int32_t t,
                      int32_t mode, float* part, float* amax_val, int32_t* amax_idx, float* logits);
/* Device time of the projection GEMM alone: seeded synthetic weights (tiled layout) and
 * tokens allocated internally, `iters` back-to-back launches of the production plan
 * (PDL, one CUDA graph) timed with CUDA events after one warm replay; *us_per_launch =
 * graph time / iters. mode as spin_gemm. Synchronous; for probes and the bench. */
spin_status spin_gemm_bench(int32_t n_out, int32_t k, int32_t t, int32_t mode, int32_t iters,
                            double* us_per_launch);

/* Packed ragged causal attention over a KV cache [layers][slots][heads][ctx][hd]
 * (bf16, device). q: [sum(qlen)][heads*hd] fp32 rows, request i owning qlen[i]
 * consecutive rows at positions kvlen[i]-qlen[i] .. kvlen[i]-1; the work list is
 * pack(kvlen, width). out: [sum(qlen)][heads*hd] bf16. Host arrays for the request shapes. */
spin_status spin_attention(void* stream, int32_t n_heads, int32_t head_dim, int32_t layers, int32_t slots,
                           int32_t ctx, int32_t layer, const void* k_cache, const void* v_cache, const void* q,
                           int32_t n_req, const int32_t* req_slot, const int32_t* req_qlen, const int32_t* req_kvlen,
                           int32_t width, void* out);
/* The same production kernel family with an explicit score scale and causal flag:
 * scale = 1, causal = 0 is the reference's toy mode (attention.cpp:67-162: unscaled,
 * every query sees all of its request's keys; kvlen may then be < qlen). Used by
 * tests/test_gpu_attention_toy.py to pin the production kernel to the reference's
 * own reference_attention / decomposed_attention outputs. */
spin_status spin_attention_ex(void* stream, int32_t n_heads, int32_t head_dim, int32_t layers, int32_t slots,
                              int32_t ctx, int32_t layer, const void* k_cache, const void* v_cache, const void* q,
                              int32_t n_req, const int32_t* req_slot, const int32_t* req_qlen,
                              const int32_t* req_kvlen, int32_t width, float scale, int32_t causal, void* out);

#ifdef __cplusplus
}
#endif

#endif /* SPIN_C_H_ */
