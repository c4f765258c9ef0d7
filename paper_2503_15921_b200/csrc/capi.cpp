// extern "C" entry points of libspin.so (declared in include/spin_c.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "engine.hpp"
#include "gemm.cuh"
#include "kernels.cuh"
#include "pack.hpp"
#include "spin_c.h"
#include "status.hpp"

namespace spin {
namespace {
thread_local std::string g_last_error;
int num_sms_cached() {
  static int n = [] {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
  }();
  return n;
}

// Device allocations released at scope exit (kernel-level entry points).
struct DevAllocs {
  std::vector<void*> ptrs;
  void* get(size_t bytes) {
    void* p = nullptr;
    check_cuda(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "malloc");
    ptrs.push_back(p);
    return p;
  }
  ~DevAllocs() {
    for (void* p : ptrs) cudaFree(p);
  }
};

// Per-forward metadata of an extend-mode meta launch over n_req requests
// packed into `rows` pack rows with `chunks` attention chunks per row.
FwdMeta alloc_meta(DevAllocs& A, int n_req, int rows, int chunks) {
  const int seg_cap = n_req + rows;
  const int piece_cap = seg_cap + rows * chunks;
  FwdMeta m{};
  m.req_slot = static_cast<int32_t*>(A.get(4 * n_req));
  m.req_qstart = static_cast<int32_t*>(A.get(4 * n_req));
  m.req_qlen = static_cast<int32_t*>(A.get(4 * n_req));
  m.req_kvlen = static_cast<int32_t*>(A.get(4 * n_req));
  m.seg = static_cast<int32_t*>(A.get(20 * seg_cap));
  m.row_ptr = static_cast<int32_t*>(A.get(4 * (rows + 1)));
  m.row_len = static_cast<int32_t*>(A.get(4 * rows));
  m.row_seg = static_cast<int32_t*>(A.get(4 * seg_cap));
  m.req_seg0 = static_cast<int32_t*>(A.get(4 * n_req));
  m.req_nseg = static_cast<int32_t*>(A.get(4 * n_req));
  m.n_seg = static_cast<int32_t*>(A.get(8));
  m.item_ptr = static_cast<int32_t*>(A.get(4 * (rows * chunks + 1)));
  m.pieces = static_cast<int32_t*>(A.get(64 * static_cast<size_t>(piece_cap)));
  m.req_pptr = static_cast<int32_t*>(A.get(4 * (n_req + 1)));
  m.req_plist = static_cast<int32_t*>(A.get(4 * static_cast<size_t>(piece_cap)));
  m.n_pieces = static_cast<int32_t*>(A.get(4));
  m.err = static_cast<int32_t*>(A.get(4));
  check_cuda(zero_sync(m.err, 4), "memset");
  m.piece_cap = piece_cap;
  return m;
}

void check_meta_status(const FwdMeta& m, const char* who) {
  int32_t e = 0;
  check_cuda(cudaMemcpy(&e, m.err, 4, cudaMemcpyDeviceToHost), "d2h status");
  if (e != 0) fail(SPIN_CAPACITY_ERROR, std::string(who) + ": attention work list exceeds its buffers");
}
}  // namespace
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace spin

using namespace spin;

extern "C" {

int spin_abi_version(void) { return SPIN_ABI_VERSION; }
const char* spin_last_error(void) { return g_last_error.c_str(); }

spin_status spin_pack(const int32_t* kv_lens, int32_t n, int32_t width, int32_t* length, int32_t* rows,
                      spin_segment* segments, int32_t seg_cap, int32_t* n_segments, int64_t* padding_tokens,
                      int32_t* q_replica_rows) {
  return guarded([&] {
    if (n < 0 || (n > 0 && kv_lens == nullptr)) fail(SPIN_INPUT_ERROR, "spin_pack: bad input arrays");
    const PackResult p = pack_lengths(kv_lens, n, width);
    if (static_cast<int32_t>(p.segments.size()) > seg_cap)
      fail(SPIN_SIZE_ERROR, "spin_pack: segment buffer too small");
    if (length) *length = p.length;
    if (rows) *rows = p.rows;
    if (n_segments) *n_segments = static_cast<int32_t>(p.segments.size());
    if (padding_tokens) *padding_tokens = p.padding;
    if (segments && !p.segments.empty())
      std::memcpy(segments, p.segments.data(), p.segments.size() * sizeof(spin_segment));
    if (q_replica_rows && n > 0) std::memcpy(q_replica_rows, p.q_replica_rows.data(), n * sizeof(int32_t));
  });
}

spin_status spin_naive_padding(const int32_t* kv_lens, int32_t n, int64_t* padding) {
  return guarded([&] { *padding = naive_padding_of(kv_lens, n); });
}

spin_status spin_verify_batch_cost(const int32_t* kv_lens, int32_t n, int32_t window, int32_t packing,
                                   int32_t pack_width, int64_t* tokens, int64_t* padding) {
  return guarded([&] {
    const VerifyCost c = verify_cost(kv_lens, n, window, packing != 0, pack_width);
    *tokens = c.tokens;
    *padding = c.padding;
  });
}

spin_status spin_gemm_info(int32_t n_out, int32_t k, int32_t t, int32_t mode, int32_t* max_pieces, int32_t* grid,
                           int32_t* bn) {
  return guarded([&] {
    if (n_out < 1 || k < 1 || t < 1) fail(SPIN_INPUT_ERROR, "spin_gemm_info: empty shape");
    const GemmPlan p = gemm_plan(n_out, k, t, mode, num_sms_cached());
    if (max_pieces) *max_pieces = p.max_pieces;
    if (grid) *grid = p.grid;
    if (bn) *bn = p.bn;
  });
}

spin_status spin_gemm(void* stream, const void* w, const void* x, int32_t n_out, int32_t k, int32_t t, int32_t mode,
                      float* part, float* amax_val, int32_t* amax_idx, float* logits) {
  return guarded([&] {
    if (n_out < 1 || k < 1 || t < 1) fail(SPIN_INPUT_ERROR, "spin_gemm: empty shape");
    if (k % 8 != 0) fail(SPIN_INPUT_ERROR, "spin_gemm: K must be a multiple of 8 (16-B rows)");
    const GemmPlan p = gemm_plan(n_out, k, t, mode, num_sms_cached());
    // row-major caller weights -> the tiled GEMM layout
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    void* wt = nullptr;
    check_cuda(cudaMalloc(&wt, tiled_weight_elems(n_out, k) * 2), "malloc");
    launch_tile_weights(static_cast<const bf16*>(w), static_cast<bf16*>(wt), n_out, k, st);
    GemmEpilogue e;
    e.mode = mode;
    e.part = part;
    e.amax_val = amax_val;
    e.amax_idx = amax_idx;
    e.logits = logits;
    if (mode == kGemmPartial && part == nullptr) fail(SPIN_INPUT_ERROR, "spin_gemm: partial buffer missing");
    if (mode == kGemmArgmax && (amax_val == nullptr || amax_idx == nullptr))
      fail(SPIN_INPUT_ERROR, "spin_gemm: argmax buffers missing");
    const cudaError_t err = gemm_launch(p, wt, x, e, st, false);
    const cudaError_t err2 = cudaStreamSynchronize(st);
    cudaFree(wt);
    check_cuda(err, "gemm launch");
    check_cuda(err2, "gemm");
  });
}


spin_status spin_gemm_bench(int32_t n_out, int32_t k, int32_t t, int32_t mode, int32_t iters,
                            double* us_per_launch) {
  return guarded([&] {
    if (n_out < 1 || k < 1 || t < 1 || iters < 1) fail(SPIN_INPUT_ERROR, "spin_gemm_bench: empty shape");
    if (k % 8 != 0) fail(SPIN_INPUT_ERROR, "spin_gemm_bench: K must be a multiple of 8 (16-B rows)");
    if (us_per_launch == nullptr) fail(SPIN_INPUT_ERROR, "spin_gemm_bench: null output");
    const GemmPlan p = gemm_plan(n_out, k, t, mode, num_sms_cached());
    bf16 *w = nullptr, *x = nullptr;
    float *out = nullptr, *logits = nullptr;
    int32_t* idx = nullptr;
    const size_t out_elems = mode == kGemmPartial ? static_cast<size_t>(p.max_pieces) * t * n_out
                                                  : static_cast<size_t>(p.n_mtiles) * t;
    cudaStream_t st = nullptr;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    cudaEvent_t a = nullptr, b = nullptr;
    auto cleanup = [&] {
      if (ge) cudaGraphExecDestroy(ge);
      if (g) cudaGraphDestroy(g);
      if (a) cudaEventDestroy(a);
      if (b) cudaEventDestroy(b);
      if (st) cudaStreamDestroy(st);
      cudaFree(w), cudaFree(x), cudaFree(out), cudaFree(idx), cudaFree(logits);
    };
    try {
      check_cuda(cudaMalloc(&w, tiled_weight_elems(n_out, k) * 2), "malloc");
      check_cuda(cudaMalloc(&x, static_cast<size_t>(t) * k * 2), "malloc");
      check_cuda(cudaMalloc(&out, out_elems * 4), "malloc");
      check_cuda(cudaMalloc(&idx, out_elems * 4), "malloc");
      check_cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
      // tiled layout of seeded weights is still a weight matrix (values do not matter for timing)
      launch_init_weights(w, n_out, k, 0x5350494eull, 0.05f, nullptr, 0.f, 1, 0, 0, 0u, 1, st);
      launch_init_weights(x, t, k, 0x58ull, 1.f, nullptr, 0.f, 1, 0, 0, 0u, 0, st);
      GemmEpilogue e;
      e.mode = mode;
      e.part = out;
      e.amax_val = out;
      e.amax_idx = idx;
      check_cuda(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "capture");
      for (int i = 0; i < iters; ++i) check_cuda(gemm_launch(p, w, x, e, st, true), "gemm launch");
      check_cuda(cudaStreamEndCapture(st, &g), "capture");
      check_cuda(cudaGraphInstantiate(&ge, g, 0), "instantiate");
      check_cuda(cudaEventCreate(&a), "event");
      check_cuda(cudaEventCreate(&b), "event");
      check_cuda(cudaGraphLaunch(ge, st), "graph");
      check_cuda(cudaEventRecord(a, st), "event");
      check_cuda(cudaGraphLaunch(ge, st), "graph");
      check_cuda(cudaEventRecord(b, st), "event");
      check_cuda(cudaEventSynchronize(b), "gemm bench");
      float ms = 0.f;
      check_cuda(cudaEventElapsedTime(&ms, a, b), "event");
      *us_per_launch = 1e3 * ms / iters;
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

// ---------------------------------------------------------------- attention operator
spin_status spin_reference_attention(int32_t q_rows, int32_t kv_rows, int32_t dim, const double* q, const double* k,
                                     const double* v, double* out) {
  if (kv_rows == 0) {
    set_last_error("reference_attention: empty KV");
    return SPIN_INPUT_ERROR;
  }
  spin_segment seg{0, 0, 0, kv_rows, 0};
  return spin_decomposed_attention(1, dim, &q_rows, &kv_rows, q, k, v, &seg, 1, 1, kv_rows, nullptr, out);
}

spin_status spin_decomposed_attention(int32_t n_req, int32_t dim, const int32_t* q_rows, const int32_t* kv_rows,
                                      const double* q, const double* k, const double* v, const spin_segment* segs,
                                      int32_t n_segs, int32_t width, int32_t length, const int32_t* mask,
                                      double* out) {
  return guarded([&] {
    if (n_req < 0 || dim < 1 || n_segs < 0 || width < 0 || length < 0)
      fail(SPIN_INPUT_ERROR, "decomposed_attention: bad sizes");
    // check_layout_consistency (attention.cpp:23-63): rebuild the indicator,
    // compare with the caller's mask, and require every request's tokens be
    // covered exactly once.
    std::vector<int32_t> cells(static_cast<size_t>(width) * length, -1);
    for (int s = 0; s < n_segs; ++s) {
      const spin_segment& g = segs[s];
      if (g.row < 0 || g.row >= width || g.col_start < 0 || g.col_end > length || g.col_start >= g.col_end)
        fail(SPIN_CONSISTENCY_ERROR, "build_indicator: segment out of bounds");
      for (int c = g.col_start; c < g.col_end; ++c) {
        int32_t& cell = cells[static_cast<size_t>(g.row) * length + c];
        if (cell != -1) fail(SPIN_CONSISTENCY_ERROR, "build_indicator: overlapping segments");
        cell = g.request_id;
      }
    }
    if (mask != nullptr && std::memcmp(mask, cells.data(), cells.size() * 4) != 0)
      fail(SPIN_CONSISTENCY_ERROR, "decomposed_attention: mask does not match layout");
    std::vector<int32_t> q_off(n_req + 1, 0), kv_off(n_req + 1, 0);
    for (int i = 0; i < n_req; ++i) {
      if (q_rows[i] < 0 || kv_rows[i] < 1) fail(SPIN_INPUT_ERROR, "decomposed_attention: empty request");
      q_off[i + 1] = q_off[i] + q_rows[i];
      kv_off[i + 1] = kv_off[i] + kv_rows[i];
    }
    std::vector<char> covered(kv_off[n_req], 0);
    for (int s = 0; s < n_segs; ++s) {
      const spin_segment& g = segs[s];
      if (g.request_id < 0 || g.request_id >= n_req)
        fail(SPIN_CONSISTENCY_ERROR, "decomposed_attention: segment references unknown request");
      for (int t = 0; t < g.col_end - g.col_start; ++t) {
        const int tok = g.token_offset + t;
        if (tok >= kv_rows[g.request_id] || covered[kv_off[g.request_id] + tok])
          fail(SPIN_CONSISTENCY_ERROR, "decomposed_attention: segment tokens do not tile the request");
        covered[kv_off[g.request_id] + tok] = 1;
      }
    }
    for (char c : covered)
      if (!c) fail(SPIN_CONSISTENCY_ERROR, "decomposed_attention: request not fully packed");
    // work lists: segments grouped by row (column order) and by request
    std::vector<int32_t> seg5(static_cast<size_t>(n_segs) * 5), row_ptr(width + 1, 0), row_seg(n_segs),
        req_seg0(n_req, 0), req_nseg(n_req, 0);
    std::vector<int> order(n_segs);
    for (int s = 0; s < n_segs; ++s) {
      seg5[5 * s] = segs[s].request_id, seg5[5 * s + 1] = segs[s].row, seg5[5 * s + 2] = segs[s].col_start;
      seg5[5 * s + 3] = segs[s].col_end, seg5[5 * s + 4] = segs[s].token_offset;
      ++row_ptr[segs[s].row + 1];
      order[s] = s;
    }
    for (int r = 0; r < width; ++r) row_ptr[r + 1] += row_ptr[r];
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      return segs[a].row != segs[b].row ? segs[a].row < segs[b].row : segs[a].col_start < segs[b].col_start;
    });
    for (int s = 0; s < n_segs; ++s) row_seg[s] = order[s];
    // partials are indexed by segment id; the combine walks a request's ids
    std::vector<int32_t> by_req(n_segs);
    std::vector<int> ro(n_segs);
    for (int s = 0; s < n_segs; ++s) ro[s] = s;
    std::stable_sort(ro.begin(), ro.end(), [&](int a, int b) { return segs[a].request_id < segs[b].request_id; });
    // remap so each request's segments are contiguous ids
    std::vector<int32_t> newid(n_segs);
    for (int s = 0; s < n_segs; ++s) newid[ro[s]] = s;
    std::vector<int32_t> seg5n(seg5.size());
    for (int s = 0; s < n_segs; ++s)
      for (int f = 0; f < 5; ++f) seg5n[5 * newid[s] + f] = seg5[5 * s + f];
    for (int s = 0; s < n_segs; ++s) row_seg[s] = newid[row_seg[s]];
    for (int s = n_segs - 1; s >= 0; --s) {
      const int rq = seg5n[5 * s];
      req_seg0[rq] = s;
      ++req_nseg[rq];
    }
    int qmax = 1;
    for (int i = 0; i < n_req; ++i) qmax = std::max(qmax, q_rows[i]);
    // device buffers
    auto bytes_d = [](size_t n) { return n * sizeof(double); };
    const size_t nq = static_cast<size_t>(q_off[n_req]) * dim, nk = static_cast<size_t>(kv_off[n_req]) * dim;
    const size_t np = static_cast<size_t>(std::max(n_segs, 1)) * qmax;
    std::vector<void*> bufs;
    auto dmal = [&](size_t b) {
      void* p = nullptr;
      check_cuda(cudaMalloc(&p, std::max<size_t>(b, 8)), "cudaMalloc");
      bufs.push_back(p);
      return p;
    };
    struct Free {
      std::vector<void*>* b;
      ~Free() {
        for (void* p : *b) cudaFree(p);
      }
    } freer{&bufs};
    double* dq = static_cast<double*>(dmal(bytes_d(nq)));
    double* dk = static_cast<double*>(dmal(bytes_d(nk)));
    double* dv = static_cast<double*>(dmal(bytes_d(nk)));
    double* dout = static_cast<double*>(dmal(bytes_d(nq)));
    double* pm = static_cast<double*>(dmal(bytes_d(np)));
    double* pl = static_cast<double*>(dmal(bytes_d(np)));
    double* po = static_cast<double*>(dmal(bytes_d(np * dim)));
    int32_t* ib = static_cast<int32_t*>(dmal(4 * (3 * (n_req + 1) + seg5n.size() + row_ptr.size() + row_seg.size() +
                                                  2 * n_req + 8)));
    std::vector<int32_t> host_ints;
    auto put = [&](const std::vector<int32_t>& v) {
      const size_t o = host_ints.size();
      host_ints.insert(host_ints.end(), v.begin(), v.end());
      return ib + o;
    };
    std::vector<int32_t> qr(q_rows, q_rows + n_req);
    const int32_t* d_qoff = put(q_off);
    const int32_t* d_kvoff = put(kv_off);
    const int32_t* d_qrows = put(qr);
    const int32_t* d_seg = put(seg5n);
    const int32_t* d_rowptr = put(row_ptr);
    const int32_t* d_rowseg = put(row_seg);
    const int32_t* d_s0 = put(req_seg0);
    const int32_t* d_ns = put(req_nseg);
    check_cuda(upload_sync(ib, host_ints.data(), host_ints.size() * 4), "h2d");
    check_cuda(upload_sync(dq, q, bytes_d(nq)), "h2d");
    check_cuda(upload_sync(dk, k, bytes_d(nk)), "h2d");
    check_cuda(upload_sync(dv, v, bytes_d(nk)), "h2d");
    launch_toy_attention(dq, dk, dv, d_qoff, d_kvoff, d_qrows, d_seg, n_segs, d_rowptr, d_rowseg, width, d_s0, d_ns,
                         n_req, dim, qmax, pm, pl, po, dout, nullptr);
    check_cuda(cudaGetLastError(), "toy attention");
    check_cuda(cudaMemcpy(out, dout, bytes_d(nq), cudaMemcpyDeviceToHost), "d2h");
  });
}

// ---------------------------------------------------------------- engine
struct spin_ctx {
  std::unique_ptr<Engine> eng;
};

spin_status spin_ctx_create(const spin_model_desc* target, const spin_model_desc* ssms, int32_t n_ssm,
                            const spin_engine_opts* opts, spin_ctx** out) {
  return guarded([&] {
    if (!target || !ssms || !opts || !out) fail(SPIN_INPUT_ERROR, "spin_ctx_create: null argument");
    auto ctx = std::make_unique<spin_ctx>();
    ctx->eng = std::make_unique<Engine>(*target, ssms, n_ssm, *opts);
    *out = ctx.release();
  });
}

spin_status spin_ctx_destroy(spin_ctx* ctx) {
  return guarded([&] { delete ctx; });
}

spin_status spin_prefill(spin_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* prompt_lens,
                         const int32_t* prompts) {
  return guarded([&] {
    if (!ctx) fail(SPIN_INPUT_ERROR, "null ctx");
    ctx->eng->prefill(n, slots, prompt_lens, prompts);
  });
}

spin_status spin_round(spin_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* ssm_of, spin_round_out* out) {
  return guarded([&] {
    if (!ctx) fail(SPIN_INPUT_ERROR, "null ctx");
    ctx->eng->round(n, slots, ssm_of, nullptr, out);
  });
}

spin_status spin_set_micro_batches(spin_ctx* ctx, const int32_t* per_ssm, int32_t n_ssm) {
  return guarded([&] {
    if (!ctx || !per_ssm) fail(SPIN_INPUT_ERROR, "spin_set_micro_batches: null argument");
    ctx->eng->set_micro_batches(per_ssm, n_ssm);
  });
}

spin_status spin_get_micro_batches(spin_ctx* ctx, int32_t* per_ssm, int32_t n_ssm) {
  return guarded([&] {
    if (!ctx || !per_ssm) fail(SPIN_INPUT_ERROR, "spin_get_micro_batches: null argument");
    ctx->eng->get_micro_batches(per_ssm, n_ssm);
  });
}

spin_status spin_tune_micro_batches(spin_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* ssm_of,
                                    int32_t max_micro_batches, int32_t probe_rounds, double threshold,
                                    int32_t* chosen, double* curve, int32_t curve_cap, int32_t* n_curve) {
  return guarded([&] {
    if (!ctx || !slots || !ssm_of) fail(SPIN_INPUT_ERROR, "spin_tune_micro_batches: null argument");
    int nc = 0;
    ctx->eng->tune_micro_batches(n, slots, ssm_of, max_micro_batches, probe_rounds, threshold, chosen, curve,
                                 curve_cap, &nc);
    if (n_curve) *n_curve = nc;
  });
}

spin_status spin_round_prewarm(spin_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* ssm_of,
                               const int32_t* prewarm, spin_round_out* out) {
  return guarded([&] {
    if (!ctx) fail(SPIN_INPUT_ERROR, "null ctx");
    ctx->eng->round(n, slots, ssm_of, prewarm, out);
  });
}

spin_status spin_run_rounds(spin_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* ssm_of, int32_t rounds,
                            int64_t* emitted, float* device_ms) {
  return guarded([&] {
    if (!ctx) fail(SPIN_INPUT_ERROR, "null ctx");
    ctx->eng->run_rounds(n, slots, ssm_of, rounds, emitted, device_ms);
  });
}

spin_status spin_read_tokens(spin_ctx* ctx, int32_t slot, int32_t* tokens, int32_t cap, int32_t* len) {
  return guarded([&] {
    if (!ctx) fail(SPIN_INPUT_ERROR, "null ctx");
    ctx->eng->read_tokens(slot, tokens, cap, len);
  });
}

spin_status spin_read_logits(spin_ctx* ctx, float* logits, int64_t cap, int32_t* rows) {
  return guarded([&] {
    if (!ctx) fail(SPIN_INPUT_ERROR, "null ctx");
    ctx->eng->read_logits(logits, cap, rows);
  });
}

spin_status spin_profile_round(spin_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* ssm_of, double* ms,
                               double* bytes, int64_t* launches) {
  return guarded([&] {
    if (!ctx) fail(SPIN_INPUT_ERROR, "null ctx");
    ctx->eng->profile_round(n, slots, ssm_of, ms, bytes, launches);
  });
}

spin_status spin_round_launches(spin_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* ssm_of,
                                int64_t* launches) {
  return guarded([&] {
    if (!ctx) fail(SPIN_INPUT_ERROR, "null ctx");
    *launches = ctx->eng->launches_per_round(n, slots, ssm_of);
  });
}

spin_status spin_kernel_bench(spin_ctx* ctx, int32_t kind, int32_t iters, double* us_per_launch,
                              double* bytes_per_launch) {
  return guarded([&] {
    if (!ctx) fail(SPIN_INPUT_ERROR, "null ctx");
    ctx->eng->kernel_bench(kind, iters, us_per_launch, bytes_per_launch);
  });
}

spin_status spin_verify_bench(spin_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* draft_lens,
                              const int32_t* drafts, int32_t packed, int32_t iters, spin_verify_stats* out) {
  return guarded([&] {
    if (!ctx) fail(SPIN_INPUT_ERROR, "null ctx");
    if (!slots || !draft_lens) fail(SPIN_INPUT_ERROR, "verify_bench: null arrays");
    ctx->eng->verify_bench(n, slots, draft_lens, drafts, packed, iters, out);
  });
}

spin_status spin_last_round_trace(spin_ctx* ctx, float* spec_end_ms, int32_t cap) {
  return guarded([&] {
    if (!ctx || !spec_end_ms) fail(SPIN_INPUT_ERROR, "last_round_trace: null argument");
    ctx->eng->last_round_trace(spec_end_ms, cap);
  });
}

spin_status spin_switch_ssm(spin_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* ssm_of) {
  return guarded([&] {
    if (!ctx) fail(SPIN_INPUT_ERROR, "null ctx");
    (void)ctx->eng->switch_ssm(n, slots, ssm_of);
  });
}


// Kernel-level entry for the packed ragged causal attention (device pointers).
// The work list is built on the device by the same meta kernel the engine uses
// (request decomposition in extend mode: requests uploaded by the host).
spin_status spin_attention(void* stream, int32_t n_heads, int32_t head_dim, int32_t layers, int32_t slots,
                           int32_t ctx, int32_t layer, const void* k_cache, const void* v_cache, const void* q,
                           int32_t n_req, const int32_t* req_slot, const int32_t* req_qlen, const int32_t* req_kvlen,
                           int32_t width, void* out) {
  return spin_attention_ex(stream, n_heads, head_dim, layers, slots, ctx, layer, k_cache, v_cache, q, n_req, req_slot,
                           req_qlen, req_kvlen, width, static_cast<float>(1.0 / std::sqrt(double(head_dim))), 1, out);
}

spin_status spin_attention_ex(void* stream, int32_t n_heads, int32_t head_dim, int32_t layers, int32_t slots,
                              int32_t ctx, int32_t layer, const void* k_cache, const void* v_cache, const void* q,
                              int32_t n_req, const int32_t* req_slot, const int32_t* req_qlen,
                              const int32_t* req_kvlen, int32_t width, float scale, int32_t causal, void* out) {
  return guarded([&] {
    if (head_dim != 64 && head_dim != 128) fail(SPIN_INPUT_ERROR, "spin_attention: head_dim must be 64 or 128");
    if (n_req < 1 || n_req > 1024) fail(SPIN_INPUT_ERROR, "spin_attention: batch must be 1..1024 requests");
    int qmax = 1;
    std::vector<int32_t> qstart(n_req);
    int T = 0;
    for (int i = 0; i < n_req; ++i) {
      if (req_qlen[i] < 1 || req_qlen[i] > 17 || req_kvlen[i] < 1 || req_kvlen[i] > ctx ||
          (causal && req_kvlen[i] < req_qlen[i]))
        fail(SPIN_INPUT_ERROR, "spin_attention: bad request shape");
      if (req_slot[i] < 0 || req_slot[i] >= slots) fail(SPIN_INPUT_ERROR, "spin_attention: slot out of range");
      qstart[i] = T;
      T += req_qlen[i];
      qmax = std::max(qmax, req_qlen[i]);
    }
    int dev = 0, sms = 148;
    check_cuda(cudaGetDevice(&dev), "device");
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int rows = width > 0 ? std::min<int>(width, n_req) : n_req;
    const int chunks = attn_chunks(rows, n_heads, sms);
    DevAllocs allocs;
    FwdMeta m = alloc_meta(allocs, n_req, rows, chunks);
    const int piece_cap = m.piece_cap;
    auto dal = [&](size_t bytes) { return allocs.get(bytes); };
    const int qpad = 8 * ((qmax + 7) / 8);
    const size_t np = static_cast<size_t>(piece_cap) * n_heads * qpad;
    AttnWork w{};
    w.part_m = static_cast<float*>(dal(4 * np));
    w.part_l = static_cast<float*>(dal(4 * np));
    w.part_o = static_cast<float*>(dal(4 * np * head_dim));
    w.counter = static_cast<int32_t*>(dal(4 * static_cast<size_t>(n_req) * n_heads));
    w.qmax = qmax;
    w.chunks = chunks;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    check_cuda(cudaMemsetAsync(w.counter, 0, 4 * static_cast<size_t>(n_req) * n_heads, s), "memset");
    check_cuda(cudaMemcpyAsync(m.req_slot, req_slot, 4 * n_req, cudaMemcpyHostToDevice, s), "h2d");
    check_cuda(cudaMemcpyAsync(m.req_qstart, qstart.data(), 4 * n_req, cudaMemcpyHostToDevice, s), "h2d");
    check_cuda(cudaMemcpyAsync(m.req_qlen, req_qlen, 4 * n_req, cudaMemcpyHostToDevice, s), "h2d");
    check_cuda(cudaMemcpyAsync(m.req_kvlen, req_kvlen, 4 * n_req, cudaMemcpyHostToDevice, s), "h2d");
    MetaArgs a{};
    a.mode = kMetaExtend;
    a.n_req = n_req;
    a.width = rows;
    a.chunks = chunks;
    SlotState st{};
    launch_meta(a, st, m, s);
    // caller caches are in the standard [..][ctx][hd] layout: swizzled copies (kv_swz) + 16 padding rows
    const int64_t kv_rows = static_cast<int64_t>(layers) * slots * n_heads * ctx;
    bf16* ks = static_cast<bf16*>(dal((kv_rows + 16) * head_dim * 2));
    bf16* vs = static_cast<bf16*>(dal((kv_rows + 16) * head_dim * 2));
    launch_swizzle_kv(static_cast<const bf16*>(k_cache), ks, kv_rows, head_dim, ctx, s);
    launch_swizzle_kv(static_cast<const bf16*>(v_cache), vs, kv_rows, head_dim, ctx, s);
    AttnGeom g{n_heads, head_dim, slots, ctx, layer, scale, ks, vs};
    g.causal = causal != 0;
    CUtensorMap tk{}, tv{};  // unused by the bulk-copy attention
    launch_attention(tk, tv, m, rows, n_req, g, static_cast<const float*>(q), w, static_cast<bf16*>(out), s);
    check_cuda(cudaGetLastError(), "attention launch");
    check_cuda(cudaStreamSynchronize(s), "attention");
    check_meta_status(m, "spin_attention");
  });
}

// ---------------------------------------------------------------- device plumbing
// Torch-free device memory for callers and tests (the product needs no framework).
spin_status spin_device_count(int32_t* count) {
  if (!count) {
    set_last_error("spin_device_count: null argument");
    return SPIN_INPUT_ERROR;
  }
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  *count = e == cudaSuccess ? n : 0;
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    set_last_error(std::string("no CUDA device: ") + cudaGetErrorString(e));
  } else {
    set_last_error("");
  }
  return SPIN_OK;
}

spin_status spin_device_alloc(int32_t device, size_t bytes, void** ptr) {
  return guarded([&] {
    if (!ptr) fail(SPIN_INPUT_ERROR, "spin_device_alloc: null argument");
    check_cuda(cudaSetDevice(device), "cudaSetDevice");
    check_cuda(cudaMalloc(ptr, std::max<size_t>(bytes, 16)), "cudaMalloc");
    check_cuda(zero_sync(*ptr, std::max<size_t>(bytes, 16)), "cudaMemset");
  });
}

spin_status spin_device_free(void* ptr) {
  return guarded([&] { check_cuda(cudaFree(ptr), "cudaFree"); });
}

spin_status spin_memcpy(void* dst, const void* src, size_t bytes, int32_t kind) {
  return guarded([&] {
    if (kind < 1 || kind > 3) fail(SPIN_INPUT_ERROR, "spin_memcpy: kind must be 1 (H2D), 2 (D2H) or 3 (D2D)");
    const cudaMemcpyKind k = kind == 1 ? cudaMemcpyHostToDevice : kind == 2 ? cudaMemcpyDeviceToHost
                                                                           : cudaMemcpyDeviceToDevice;
    if (bytes == 0) return;
    if (k == cudaMemcpyHostToDevice) {  // complete before return, whatever stream reads it next
      check_cuda(upload_sync(dst, src, bytes), "cudaMemcpy");
    } else {
      check_cuda(cudaMemcpy(dst, src, bytes, k), "cudaMemcpy");
      if (k == cudaMemcpyDeviceToDevice) check_cuda(cudaDeviceSynchronize(), "cudaMemcpy");  // D2D is asynchronous
    }
  });
}

// Device request decomposition (the meta kernel's packer, kernels.cu) on its own:
// same contract as spin_pack, computed on the GPU; used to pin the device packer
// to the reference goldens (packing.cpp:16-103).
spin_status spin_pack_device(const int32_t* kv_lens, int32_t n, int32_t width, int32_t* length, int32_t* rows,
                             spin_segment* segments, int32_t seg_cap, int32_t* n_segments, int64_t* padding_tokens,
                             int32_t* q_replica_rows) {
  return guarded([&] {
    if (n < 0 || (n > 0 && kv_lens == nullptr)) fail(SPIN_INPUT_ERROR, "spin_pack_device: bad input arrays");
    // validation and error taxonomy identical to the host packer (pack.cpp)
    pack_validate(kv_lens, n, width);
    if (n == 0) {
      if (length) *length = 0;
      if (rows) *rows = 0;
      if (n_segments) *n_segments = 0;
      if (padding_tokens) *padding_tokens = 0;
      return;
    }
    if (n > 1024) fail(SPIN_SIZE_ERROR, "spin_pack_device: at most 1024 requests per pack");
    const int nrows = std::min<int>(width, n);
    DevAllocs allocs;
    FwdMeta m = alloc_meta(allocs, n, nrows, 1);
    std::vector<int32_t> ones(n, 1), qs(n), zeros(n, 0);
    for (int i = 0; i < n; ++i) qs[i] = i;
    check_cuda(upload_sync(m.req_slot, zeros.data(), 4 * n), "h2d");
    check_cuda(upload_sync(m.req_qstart, qs.data(), 4 * n), "h2d");
    check_cuda(upload_sync(m.req_qlen, ones.data(), 4 * n), "h2d");
    check_cuda(upload_sync(m.req_kvlen, kv_lens, 4 * n), "h2d");
    MetaArgs a{};
    a.mode = kMetaExtend;
    a.n_req = n;
    a.width = nrows;
    a.chunks = 1;
    SlotState st{};
    launch_meta(a, st, m, nullptr);
    check_cuda(cudaGetLastError(), "meta launch");
    check_cuda(cudaDeviceSynchronize(), "meta");
    check_meta_status(m, "spin_pack_device");
    int32_t ns[2] = {0, 0};
    check_cuda(cudaMemcpy(ns, m.n_seg, 8, cudaMemcpyDeviceToHost), "d2h");
    if (ns[0] > seg_cap) fail(SPIN_SIZE_ERROR, "spin_pack_device: segment buffer too small");
    std::vector<int32_t> seg(static_cast<size_t>(ns[0]) * 5), nseg(n);
    check_cuda(cudaMemcpy(seg.data(), m.seg, seg.size() * 4, cudaMemcpyDeviceToHost), "d2h");
    check_cuda(cudaMemcpy(nseg.data(), m.req_nseg, 4 * n, cudaMemcpyDeviceToHost), "d2h");
    int64_t total = 0;
    for (int i = 0; i < n; ++i) total += kv_lens[i];
    if (length) *length = ns[1];
    if (rows) *rows = nrows;
    if (n_segments) *n_segments = ns[0];
    if (padding_tokens) *padding_tokens = static_cast<int64_t>(nrows) * ns[1] - total;
    if (segments) std::memcpy(segments, seg.data(), seg.size() * 4);
    if (q_replica_rows) std::memcpy(q_replica_rows, nseg.data(), 4 * n);
  });
}

}  // extern "C"
