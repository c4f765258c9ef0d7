// Memory-bound kernels of the verification / draft forward pass and the
// device-side bookkeeping (request decomposition, acceptance, KV rollback).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "gemm.cuh"

namespace spin {

using bf16 = __nv_bfloat16;

constexpr int kMaxSsm = 8;

// Per-forward metadata (device pointers). Rows are the token rows of the
// forward; requests own a contiguous range of rows (their queries); segments
// are the request-decomposition work items of the packed attention.
struct FwdMeta {
  int32_t* row_tok;   // [T]
  int32_t* row_slot;  // [T]  KV slot, -1: padding row (no KV write)
  int32_t* row_pos;   // [T]  absolute position
  int32_t* req_slot;  // [R]
  int32_t* req_qstart;
  int32_t* req_qlen;
  int32_t* req_kvlen;  // keys visible to the last query = last position + 1
  int32_t* seg;        // [S][5] request, row, col_start, col_end, token_offset (pack order)
  int32_t* row_ptr;    // [W+1] CSR over pack rows into row_seg
  int32_t* row_len;    // [W] used columns of each pack row
  // attention work (meta_kernel): pack row r, chunk c -> pieces [item_ptr[r*nch+c], item_ptr[r*nch+c+1])
  int32_t* item_ptr;   // [rows * nch + 1]
  int32_t* pieces;     // [P][16] {request, slot, token0, len | qstart, qlen, kvlen, pieces of request | merge-list start}
  int32_t* req_pptr;   // [R + 1] CSR: each request's pieces in (segment, chunk) = token order
  int32_t* req_plist;  // [P]
  int32_t* n_pieces;   // [1]
  int32_t piece_cap;   // capacity of pieces (and of the split-KV partial slots)
  int32_t* row_seg;    // [S] segment ids grouped by pack row, column order
  int32_t* req_seg0;   // [R] first segment (segments of a request are contiguous)
  int32_t* req_nseg;   // [R]
  int32_t* n_seg;      // [2] segment count, pack length L (packing.hpp PackedLayout::length)
  int32_t* err;        // [1] sticky device status: 1 = attention piece buffer overflow (the host
                       //     reads it back with the outcome and raises SPIN_CAPACITY_ERROR)
};

// Persistent per-slot state on the device.
struct SlotState {
  int32_t* tokens;     // [slots][ctx] committed token history
  int32_t* committed;  // [slots]
  int32_t* ssm_len;    // [n_ssm][slots] valid KV positions of each SSM cache
  int32_t* drafts;     // [slots][window]
  int32_t slots, ctx, window, n_ssm;
};

enum MetaMode : int {
  kMetaVerify = 0,   // rows: pending token + window drafts per request
  kMetaDraft0 = 1,   // rows: last two committed tokens per request
  kMetaDraftK = 2,   // rows: previous draft; collects previous step's argmax first
  kMetaCollect = 3,  // only collects the final draft step's argmax
  kMetaExtend = 4,   // rows/requests uploaded by the host; only packs
};

struct MetaArgs {
  int mode;
  int n_req;
  const int32_t* list;  // [n_req] request slots in batch order
  int step;             // draft step k (DraftK / Collect: step whose draft is collected = step-1)
  int ssm;              // SSM index for ssm_len bookkeeping
  int width;            // pack width (0: n_req)
  int padded;           // 1: one row per request padded to the longest (no decomposition)
  // previous lm_head argmax (DraftK / Collect)
  const float* amax_val;
  const int32_t* amax_idx;
  int amax_tiles;
  int prev_t;     // rows of the previous forward
  int prev_qlen;  // rows per request in the previous forward
  int chunks;     // attention chunks per pack row (attn_chunks)
};

struct LayerW {
  const bf16 *qkv, *o, *gu, *dn;
  const bf16 *sqkv = nullptr, *so = nullptr, *sgu = nullptr, *sdn = nullptr;  // draft slabs (SSMs)
};

// KV cache rows are stored pre-swizzled so that a contiguous range of keys, bulk-copied
// into shared memory, is already bank-conflict free for ldmatrix: inside every 128-B
// span of a key row, 16-B chunk c of key position p sits at chunk c ^ (p % 8).
__host__ __device__ __forceinline__ int kv_swz(int pos, int d) {
  return (d & ~63) | ((((d >> 3) & 7) ^ (pos & 7)) << 3) | (d & 7);
}

struct AttnGeom {
  int n_heads, head_dim, slots, ctx, layer;
  float scale;
  bf16* k_cache;  // [layers][slots][heads][ctx][hd], rows swizzled by kv_swz (+16 padding rows at the end)
  bf16* v_cache;
  int causal = 1;  // 0: every query sees all of its request's keys (the reference's toy mode, attention.cpp:67-96)
};

void launch_meta(const MetaArgs& a, const SlotState& st, const FwdMeta& m, cudaStream_t s);
void launch_embed_norm(const bf16* emb, const FwdMeta& m, int T, int D, float eps, float* h, bf16* xn,
                       cudaStream_t s);
// one-wave grids of the epilogue kernels (SPIN_STAMPS slot sizes)
int qkv_epilogue_blocks(int T, int D);
int swiglu_blocks(int T, int F);
void launch_qkv_epilogue(const float* part, const PieceMap& pm, const FwdMeta& m, int T, const AttnGeom& g,
                         const float* rcos, const float* rsin, float* q, cudaStream_t s,
                         unsigned long long* st = nullptr);
void launch_resid_norm(const float* part, const PieceMap& pm, int T, int D, float eps, float* h, bf16* xn,
                       cudaStream_t s, unsigned long long* st = nullptr);
void launch_swiglu(const float* part, const PieceMap& pm, int T, int F, bf16* act, cudaStream_t s,
                   unsigned long long* st = nullptr);

// Fused projections of the draft step (draft.cu): one CTA per 16/32 output rows over
// the full K, epilogue in the projection, RMSNorm folded into the consumers through
// per-unit sums of squares ssp[t][unit].
constexpr int kDraftMaxT = 32;
enum DraftProjMode : int { kDpQkv = 0, kDpGateUp = 1, kDpResid = 2 };
struct DraftProj {
  int mode;
  const bf16* w;  // slab weights (launch_slab_weights), n_out x K
  int n_out, K, T;
  float* h;            // RESID: fp32 residual stream, updated
  bf16* hb;            // RESID: bf16 copy of the updated residual (the norm consumers' token operand)
  const float* ssp;    // QKV / GATE_UP: [T][n_ssp] sums of squares of h
  int n_ssp;
  float eps;
  const bf16* x;       // bf16 token operand [T][K]: attention out / SwiGLU out / bf16(h) for QKV, GATE_UP
  float* ssp_out;      // RESID: [T][n_out / 16]
  float* q;            // QKV: fp32 [T][D], RoPE applied; K/V appended to g's caches
  AttnGeom g;
  const int32_t* row_slot;
  const int32_t* row_pos;
  const float* rcos;
  const float* rsin;
  bf16* act;           // GATE_UP: SwiGLU output [T][n_out / 2]
  unsigned long long* st;  // optional timeline stamps [CTA][4] (SPIN_STAMPS)
};
int draft_proj_units(const DraftProj& a);
// Slab copy of a tiled weight matrix for the draft projections (unit-contiguous).
size_t draft_slab_elems(int n_out, int K);
void launch_slab_weights(const bf16* tiled, bf16* slab, int mode, int n_out, int K, int hd, cudaStream_t s);
bool draft_fused_supported(int D, int H, int hd, int F, int T);
cudaError_t launch_draft_proj(const DraftProj& a, cudaStream_t s);
void launch_embed_ss(const bf16* emb, const FwdMeta& m, int T, int D, float* h, bf16* hb, float* ssp,
                     cudaStream_t s);
void launch_norm_ss(const float* h, const float* ssp, int n_ssp, int T, int D, float eps, bf16* xn, cudaStream_t s);

// Packed ragged causal attention over the KV cache (TMA-staged tiles) and the
// shared-max combine of segment partials.
struct AttnWork {
  float* part_m;  // [pieces][H][qpad]  split-KV partials (qpad = 8 * ceil(qmax / 8))
  float* part_l;
  float* part_o;  // [pieces][H][qpad][hd]
  int32_t* counter;  // [R_cap][H] arrivals per (request, head); zero between launches
  int qmax;
  int chunks;     // chunks per pack row (must equal the MetaArgs.chunks that built the work list)
  int early = 0;  // issue K/V tiles older than the queries before the dependency wait (FwdShape::early)
  unsigned long long* st = nullptr;  // optional timeline stamps [CTA][4] (SPIN_STAMPS)
};
int attn_ctas(int n_rows, int chunks, int heads, int qmax);
// Chunks per pack row so that rows x chunks x heads warps fill the GPU.
// Requests with at most kDecodeQ queries (draft steps) use the few-query kernel.
constexpr int kDecodeQ = 2;
int attn_chunks(int rows, int heads, int num_sms, int qmax = 8);
void launch_attention(const CUtensorMap& tm_k, const CUtensorMap& tm_v, const FwdMeta& m, int n_rows, int n_req,
                      const AttnGeom& g, const float* q, const AttnWork& w, bf16* out, cudaStream_t s);

void launch_accept(const FwdMeta& m, int n_req, int window, const int32_t* list, const int32_t* ssm_of_req,
                   const float* amax_val, const int32_t* amax_idx, int tiles, int T, const SlotState& st,
                   int32_t* out_accepted, int32_t* out_bonus, int32_t* out_committed, int32_t* out_drafts,
                   int32_t* out_target, unsigned long long* emitted, cudaStream_t s);

// tiled = 1: the GEMM weight layout (gemm.cuh tiled_weight_elems); 0: row-major (embedding).
// Standard-layout [rows][hd] KV rows -> the swizzled cache layout (kernel tests).
void launch_swizzle_kv(const bf16* src, bf16* dst, int64_t rows, int hd, int ctx, cudaStream_t s);
// emb/planted_g/dsize/A_inv/Cc/mask: the planted map of an lm_head (dsize = ids per domain).
void launch_init_weights(bf16* w, int64_t rows, int64_t cols, uint64_t stream, float scale, const bf16* emb,
                         float planted_g, int64_t dsize, int64_t A_inv, int64_t Cc, uint32_t mask, int tiled,
                         cudaStream_t s);
// Row-major [rows][cols] -> tiled GEMM weight layout.
void launch_tile_weights(const bf16* src, bf16* dst, int64_t rows, int64_t cols, cudaStream_t s);

// Toy-mode packed attention for the decomposed_attention operator (K/V laid
// out per request, any dim, scale 1, no causal mask).
// Computed in fp64 on the device (the reference operator is fp64).
void launch_toy_attention(const double* q, const double* k, const double* v, const int32_t* q_off,
                          const int32_t* kv_off, const int32_t* q_rows, const int32_t* seg, int n_seg,
                          const int32_t* row_ptr, const int32_t* row_seg, int n_rows, const int32_t* req_seg0,
                          const int32_t* req_nseg, int n_req, int dim, int qmax, double* part_m, double* part_l,
                          double* part_o, double* out, cudaStream_t s);

}  // namespace spin
