// Packed ragged causal attention for the verify / draft forward (K4 + K5).
//
// Work decomposition = the request decomposition of the reference packer
// (packing.cpp:16-103): pack row r holds segments (contiguous key ranges of
// one request's KV) and all rows have the same length L, so equal shares of a
// row are equal work. meta_kernel cuts every row into `chunks` column chunks
// (chosen so rows x chunks x heads ~ 8 warps per SM) and lists the pieces of
// each chunk (piece = a segment's part inside the chunk). The kernel reads the
// per-slot KV cache in place (zero-copy packing).
//
// One WARP per (row, chunk, head), no CTA-level synchronisation: the warp owns
// a ring of 16-key K/V tiles (1-D bulk copies of the pre-swizzled cache rows, lane 0 issues ahead across
// its pieces) and computes the TRANSPOSED scores S^T = K Q^T on the tensor
// cores (mma.sync m16n8k16: 16 keys are M, the request's <= 8 queries per
// n-tile are N), an online softmax per query column, and O^T += V^T P^T (head
// dims are M; P^T is re-fragmented with movmatrix). Q and P are split into
// bf16 hi + lo planes (16-bit mantissa, fp32 accumulate): scores and weights
// keep fp32-level accuracy.
//
// Combine = the shared-max aggregation of attention.cpp:128-157 in split-KV
// form: a request with several pieces writes (max, sum, unnormalised out) per
// piece; the warp that completes the last piece of a (request, head) (global
// arrival counter) merges them in token order. Deterministic run to run.
#include "kernels.cuh"
#include "ptx.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>

namespace spin {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kNW = 4;                   // warps per CTA (few-query kernel)
constexpr int kThreads = 32 * kNW;
// attn_kernel: independent warps, so CTAs of one warp let the block scheduler spread the
// (row, chunk, head) items evenly over the SMs (4-warp CTAs left 108 SMs with 8 items and
// 40 with 4 at config 2)
#ifndef SPIN_ATTN_VW
#define SPIN_ATTN_VW 1
#endif
constexpr int kVW = SPIN_ATTN_VW;
constexpr int kMaxPieces = 16;           // piece records staged per warp per pass
constexpr int kDecStages = 2;            // few-query ring depth per warp (launch_decode)
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float bf_round(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// D(16x8, fp32) += A(16x16 bf16, row) * B(16x8 bf16, col)
__device__ __forceinline__ void mma16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ uint32_t movm_t(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

// byte offset of (key row, 16-B chunk) in a 16-key tile bulk-copied from the swizzled
// cache (kv_swz): rows of HD*2 bytes, chunk c of absolute key p at c ^ (p % 8) within
// its 128-B span; `base` = absolute key of row 0 (mod 8).
template <int HD>
__device__ __forceinline__ uint32_t kvoff(int row, int chunk, int base) {
  return static_cast<uint32_t>(row * (HD * 2) + (chunk >> 3) * 128 + (((chunk & 7) ^ ((row + base) & 7)) << 4));
}

template <int HD, int NQT, int NW = kNW, int ST = 0>
struct Cfg {
  static constexpr int kWarps = NW;
  static constexpr int kStages = ST > 0 ? ST : (HD == 128 ? 3 : 4);  // per-warp ring depth
  static constexpr uint32_t kHalf = 16 * HD * 2;        // K or V of one 16-key tile
  static constexpr uint32_t kStage = 2 * kHalf;
  static constexpr uint32_t kRing = NW * kStages * kStage;
  static constexpr int kDT = HD / 16;                   // 16-dim tiles
  static constexpr int kNR = kDT * NQT * 4;             // O^T fragment registers per thread
  static constexpr int kQP = 8 * NQT;                   // padded queries
  static constexpr int kQF = kDT * NQT * 4;             // raw Q floats per thread
  static constexpr size_t kTotal = 1024 + kRing + NW * kMaxPieces * 64 + NW * kStages * 8;
};

// Piece record written by meta_kernel (FwdMeta::pieces).
struct Piece {
  int req, slot, tok0, len, qs, qlen, kvlen, npieces, pptr, pad[7];
};

// Shared-max merge of a request's split-KV partials (attention.cpp:128-157), by one warp,
// pieces in token order. Lanes own pieces for the max / sum and head dims for the
// output; every query's (max, sum) loads of all pieces are issued together, then one
// pass over the pieces accumulates up to 8 queries' outputs (independent loads).
template <int HD, int QP, bool kBatched>
__device__ __forceinline__ void merge_pieces(const FwdMeta& m, const AttnWork& w, const Piece& ph, int head, int H,
                                             int D, bf16* __restrict__ out, int lane) {
  constexpr int DV = HD / 32;  // head dims per lane
  const int npc = ph.npieces;
  if (npc > 32 || !kBatched) {  // query-serial merge: many pieces, or register-tight kernels
    for (int qi = 0; qi < ph.qlen; ++qi) {
      float M = -INFINITY;
      for (int p0 = 0; p0 < npc; p0 += 32) {
        const int pp = p0 + lane;
        const int id = pp < npc ? __ldcg(m.req_plist + ph.pptr + pp) : 0;
        const float mp = pp < npc ? __ldcg(w.part_m + (static_cast<size_t>(id) * H + head) * QP + qi) : -INFINITY;
        M = fmaxf(M, mp);
      }
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) M = fmaxf(M, __shfl_xor_sync(kFull, M, o2));
      float L = 0.f, acc[DV];
#pragma unroll
      for (int j = 0; j < DV; ++j) acc[j] = 0.f;
      for (int p0 = 0; p0 < npc; p0 += 32) {
        const int pp = p0 + lane;
        int id = 0;
        float f = 0.f;
        if (pp < npc) {
          id = __ldcg(m.req_plist + ph.pptr + pp);
          const size_t pi = (static_cast<size_t>(id) * H + head) * QP + qi;
          const float mp = __ldcg(w.part_m + pi);
          f = mp == -INFINITY ? 0.f : exp2f(mp - M);
          L += __ldcg(w.part_l + pi) * f;
        }
        const int cntp = min(32, npc - p0);
        for (int j0 = 0; j0 < cntp; ++j0) {
          const float fj = __shfl_sync(kFull, f, j0);
          const int pj = __shfl_sync(kFull, id, j0);
          if (fj == 0.f) continue;
          const float* src = w.part_o + ((static_cast<size_t>(pj) * H + head) * QP + qi) * HD + DV * lane;
#pragma unroll
          for (int j = 0; j < DV; ++j) acc[j] += __ldcg(src + j) * fj;
        }
      }
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) L += __shfl_xor_sync(kFull, L, o2);
      bf16* dst = out + static_cast<size_t>(ph.qs + qi) * D + head * HD + DV * lane;
#pragma unroll
      for (int j = 0; j < DV; ++j) dst[j] = __float2bfloat16_rn(acc[j] / L);
    }
    return;
  }
  const int pid = lane < npc ? __ldcg(m.req_plist + ph.pptr + lane) : 0;
  for (int q0 = 0; q0 < ph.qlen; q0 += 8) {
    float mq[8], lq[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const bool ok = lane < npc && q0 + i < ph.qlen;
      const size_t pi = (static_cast<size_t>(pid) * H + head) * QP + q0 + i;
      mq[i] = ok ? __ldcg(w.part_m + pi) : -INFINITY;
      lq[i] = ok ? __ldcg(w.part_l + pi) : 0.f;
    }
    float f[8], L[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float M = mq[i];
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) M = fmaxf(M, __shfl_xor_sync(kFull, M, o2));
      f[i] = mq[i] == -INFINITY ? 0.f : exp2f(mq[i] - M);
      float l = lq[i] * f[i];
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) l += __shfl_xor_sync(kFull, l, o2);
      L[i] = l;
    }
    float acc[8][DV];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < DV; ++j) acc[i][j] = 0.f;
#pragma unroll 2
    for (int pj = 0; pj < npc; ++pj) {
      const int id = __shfl_sync(kFull, pid, pj);
      const float* src = w.part_o + ((static_cast<size_t>(id) * H + head) * QP + q0) * HD + DV * lane;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float fi = __shfl_sync(kFull, f[i], pj);
        if (q0 + i >= ph.qlen || fi == 0.f) continue;
        if constexpr (HD == 128) {
          const float4 v = __ldcg(reinterpret_cast<const float4*>(src + i * HD));
          acc[i][0] += v.x * fi, acc[i][1] += v.y * fi, acc[i][2] += v.z * fi, acc[i][3] += v.w * fi;
        } else {
          const float2 v = __ldcg(reinterpret_cast<const float2*>(src + i * HD));
          acc[i][0] += v.x * fi, acc[i][1] += v.y * fi;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (q0 + i >= ph.qlen) continue;
      const float inv = 1.0f / L[i];
      bf16* dst = out + static_cast<size_t>(ph.qs + q0 + i) * D + head * HD + DV * lane;
#pragma unroll
      for (int j = 0; j < DV; ++j) dst[j] = __float2bfloat16_rn(acc[i][j] * inv);
    }
  }
}

template <int HD, int NQT>
__global__ void __launch_bounds__(32 * kVW) attn_kernel(const __grid_constant__ CUtensorMap tm_k,
                                                        const __grid_constant__ CUtensorMap tm_v, FwdMeta m,
                                                        AttnGeom g, const float* __restrict__ q, AttnWork w,
                                                        bf16* __restrict__ out, int n_items) {
  using C = Cfg<HD, NQT, kVW>;
  constexpr int S = C::kStages, DT = C::kDT, NR = C::kNR, QP = C::kQP, QF = C::kQF;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int gq = lane >> 2, cq = lane & 3;
  uint8_t* ring = smem + static_cast<size_t>(warp) * S * C::kStage;
  Piece* pcs = reinterpret_cast<Piece*>(smem + C::kRing) + warp * kMaxPieces;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::kRing + kVW * kMaxPieces * 64) + warp * S;
  const int H = g.n_heads, D = H * HD;
  const float sl2 = g.scale * kLog2e;

  const int item = blockIdx.x * kVW + warp;  // (pack row, chunk) x head, one per warp
  if (lane == 0) {
    for (int s = 0; s < S; ++s) ptx::mbar_init(&bar[s], 1);
    ptx::fence_mbar_init();
  }
  __syncwarp();
  // w.early (verify / draft forwards, where a request's only new KV rows are its query
  // positions): the work list (meta_kernel) and the KV rows older than the queries are
  // complete before this grid starts (every kernel of the chain waits on its predecessor
  // before triggering us), so pieces are staged and those K/V tiles issued BEFORE the
  // dependency wait; only q and the tiles holding this forward's new keys wait for the
  // projection kernel. Extends (virtual requests reading keys written earlier in the
  // same forward) wait first.
  const bool stamp = w.st != nullptr && threadIdx.x == 0;
  // stamps [CTA][8] (warp 0): start, wait release, first tile ready, q ready, tile loop end,
  // partial stored, merge start, end
  if (stamp) w.st[8 * blockIdx.x] = ptx::globaltimer();
  bool dep_done = false;
  if (!w.early) ptx::grid_dep_wait(), dep_done = true;
  if (item >= n_items * H) return;
  const int head = item % H, rc = item / H;
  const int p_lo = m.item_ptr[rc], p_hi = m.item_ptr[rc + 1];
  const uint64_t pol = ptx::policy_evict_first();
  const int kv_base = (g.layer * g.slots) * H;  // (kv_base + slot * H + head) * ctx + token

  int issued = 0, consumed = 0;
  for (int pb = p_lo; pb < p_hi; pb += kMaxPieces) {
    // ---- stage this warp's pieces (one 64-B record per lane)
    const int np = min(p_hi - pb, kMaxPieces);
    for (int k = lane; k < np; k += 32) {
      const int4* src = reinterpret_cast<const int4*>(m.pieces + 16 * (pb + k));
      int4* dst = reinterpret_cast<int4*>(pcs + k);
      dst[0] = src[0], dst[1] = src[1], dst[2] = src[2];
    }
    __syncwarp();
    int ik = 0, it = 0;
    auto try_issue = [&]() {
      while (issued - consumed < S && ik < np) {
        const Piece& ph = pcs[ik];
        if (it * 16 >= ph.len) {
          ++ik, it = 0;
          continue;
        }
        if (!dep_done && ph.tok0 + it * 16 + 16 > ph.kvlen - ph.qlen) break;
        if (lane == 0) {
          const int st = issued % S;
          uint8_t* dst = ring + st * C::kStage;
          const size_t r0 = (static_cast<size_t>(kv_base + ph.slot * H + head) * g.ctx) + ph.tok0 + it * 16;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          ptx::mbar_arrive_expect_tx(&bar[st], C::kStage);
          // 16 consecutive keys are one contiguous, pre-swizzled block of K and of V
          ptx::bulk_load(dst, g.k_cache + r0 * HD, C::kHalf, &bar[st], pol);
          ptx::bulk_load(dst + C::kHalf, g.v_cache + r0 * HD, C::kHalf, &bar[st], pol);
        }
        ++issued;
        ++it;
      }
    };
    try_issue();
    if (!dep_done) {
      ptx::grid_dep_wait();
      dep_done = true;
      if (stamp) w.st[8 * blockIdx.x + 1] = ptx::globaltimer();
      try_issue();
    }
    if (pb == p_lo) ptx::grid_dep_launch();  // the next GEMM takes SMs as this grid drains

    for (int k = 0; k < np; ++k) {
      const Piece ph = pcs[k];
      // Q^T fragments (B operand): thread (g, c) holds query 8nt+g, dims 16kt+2c(+1), +8(+9); hi / lo planes
      uint32_t qh[NQT][DT][2], ql[NQT][DT][2];
      {
        float qv[QF];
#pragma unroll
        for (int nt = 0; nt < NQT; ++nt) {
          const int qi = 8 * nt + gq;
          const bool ok = qi < ph.qlen;
          const float* qr = q + static_cast<size_t>(ph.qs + (ok ? qi : 0)) * D + head * HD + 2 * cq;
#pragma unroll
          for (int kt = 0; kt < DT; ++kt)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const float2 v =
                  ok ? __ldg(reinterpret_cast<const float2*>(qr + 16 * kt + 8 * hh)) : make_float2(0.f, 0.f);
              qv[((nt * DT + kt) * 2 + hh) * 2] = v.x;
              qv[((nt * DT + kt) * 2 + hh) * 2 + 1] = v.y;
            }
        }
#pragma unroll
        for (int i = 0; i < QF / 2; ++i) {
          const float x = qv[2 * i] * sl2, y = qv[2 * i + 1] * sl2;
          const float hx = bf_round(x), hy = bf_round(y);
          const int hh = i & 1, kt = (i >> 1) % DT, nt = (i >> 1) / DT;
          qh[nt][kt][hh] = pack_bf2(hx, hy);
          ql[nt][kt][hh] = pack_bf2(x - hx, y - hy);
        }
      }
      // NQT > 1: the lo plane accumulates into o (register budget); NQT = 1: separate chain
      constexpr int NRL = NQT == 1 ? NR : 1;
      float o[NR], olo[NRL];
#pragma unroll
      for (int i = 0; i < NR; ++i) o[i] = 0.f;
#pragma unroll
      for (int i = 0; i < NRL; ++i) olo[i] = 0.f;
      float mrun[NQT][2], lsum[NQT][2];
#pragma unroll
      for (int nt = 0; nt < NQT; ++nt) mrun[nt][0] = mrun[nt][1] = -INFINITY, lsum[nt][0] = lsum[nt][1] = 0.f;
      const int qbase = ph.kvlen - ph.qlen;  // absolute position of query 0
      if (stamp && k == 0 && pb == p_lo) w.st[8 * blockIdx.x + 3] = ptx::globaltimer() + (qh[0][0][0] == 12345u);

      // Software-pipelined tile loop: the scores of tile t + 1 (S^T = K Q^T, independent of
      // tile t's softmax and P V) are issued before tile t's softmax and O^T += V^T P^T, so
      // the two mma.sync chains and the exp / shuffle work of neighbouring tiles overlap
      // inside the warp (each warp owns a whole (row, head): its tile chain is the critical path).
      auto scores = [&](int stg, float (&sv)[NQT][4]) {
        // S^T = K Q^T : 16 keys x 8 queries per n-tile. Four independent accumulator
        // chains (k-step parity x hi/lo plane) keep the mma.sync pipeline full; summed at the end.
        const uint32_t kb = ptx::smem_u32(ring + stg * C::kStage);
        float sc[NQT][4][4];
#pragma unroll
        for (int nt = 0; nt < NQT; ++nt)
#pragma unroll
          for (int c = 0; c < 4; ++c) sc[nt][c][0] = sc[nt][c][1] = sc[nt][c][2] = sc[nt][c][3] = 0.f;
#pragma unroll
        for (int kt = 0; kt < DT; ++kt) {
          uint32_t a[4];
          ldsm_x4(kb + kvoff<HD>((lane & 7) + ((lane >> 3) & 1) * 8, 2 * kt + (lane >> 4), ph.tok0), a);
#pragma unroll
          for (int nt = 0; nt < NQT; ++nt) {
            mma16816(sc[nt][kt & 1], a, qh[nt][kt][0], qh[nt][kt][1]);
            mma16816(sc[nt][2 + (kt & 1)], a, ql[nt][kt][0], ql[nt][kt][1]);
          }
        }
#pragma unroll
        for (int nt = 0; nt < NQT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) sv[nt][e] = (sc[nt][0][e] + sc[nt][1][e]) + (sc[nt][2][e] + sc[nt][3][e]);
      };
      // (NQT > 1 keeps the plain order: the look-ahead scores would spill at 3 query tiles)
      constexpr bool kPipe = NQT == 1;
      const int ntile = (ph.len + 15) / 16;
      float s[NQT][4];
      if (kPipe) {
        ptx::mbar_wait(&bar[consumed % S], static_cast<uint32_t>((consumed / S) & 1));
        if (stamp && consumed == 0) w.st[8 * blockIdx.x + 2] = ptx::globaltimer();
        scores(consumed % S, s);
      }
      for (int t = 0; t < ntile; ++t) {
        const int st = consumed % S;
        const bool more = kPipe && t + 1 < ntile;
        float s_next[NQT][4];
        if (!kPipe) {
          ptx::mbar_wait(&bar[st], static_cast<uint32_t>((consumed / S) & 1));
          if (stamp && consumed == 0) w.st[8 * blockIdx.x + 2] = ptx::globaltimer();
          scores(st, s);
        }
        if (more) {  // tile t + 1 is already in flight (the ring keeps S >= 2 tiles issued ahead)
          const int st1 = (consumed + 1) % S;
          ptx::mbar_wait(&bar[st1], static_cast<uint32_t>(((consumed + 1) / S) & 1));
          scores(st1, s_next);
        }
        const uint32_t vb = ptx::smem_u32(ring + st * C::kStage) + C::kHalf;
        // ---- mask + online softmax per query column (keys gq, gq+8; queries 2cq, 2cq+1)
        const int key0 = ph.tok0 + t * 16 + gq;
        const int kend = ph.tok0 + ph.len;
        uint32_t ph_[NQT][2], pl_[NQT][2];
#pragma unroll
        for (int nt = 0; nt < NQT; ++nt) {
          float corr[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int qpos = qbase + 8 * nt + 2 * cq + e;
            const bool v0 = key0 < kend && (key0 <= qpos || !g.causal);
            const bool v1 = key0 + 8 < kend && (key0 + 8 <= qpos || !g.causal);
            s[nt][e] = v0 ? s[nt][e] : -INFINITY;
            s[nt][2 + e] = v1 ? s[nt][2 + e] : -INFINITY;
            float mx = fmaxf(s[nt][e], s[nt][2 + e]);
            mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 4));
            mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 8));
            mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 16));
            const float mnew = fmaxf(mrun[nt][e], mx);
            corr[e] = mnew == -INFINITY ? 1.f : exp2f(mrun[nt][e] - mnew);
            const float p0 = mnew == -INFINITY ? 0.f : exp2f(s[nt][e] - mnew);
            const float p1 = mnew == -INFINITY ? 0.f : exp2f(s[nt][2 + e] - mnew);
            s[nt][e] = p0;
            s[nt][2 + e] = p1;
            lsum[nt][e] = lsum[nt][e] * corr[e] + (p0 + p1);
            mrun[nt][e] = mnew;
          }
#pragma unroll
          for (int dt = 0; dt < DT; ++dt) {
            float* oo = o + (nt * DT + dt) * 4;
            oo[0] *= corr[0], oo[1] *= corr[1], oo[2] *= corr[0], oo[3] *= corr[1];
            if constexpr (NQT == 1) {
              float* ol = olo + (nt * DT + dt) * 4;
              ol[0] *= corr[0], ol[1] *= corr[1], ol[2] *= corr[0], ol[3] *= corr[1];
            }
          }
          // P^T as the B operand: movmatrix turns the (key g, queries 2c..2c+1)
          // accumulator pairs into (query g, keys 2c..2c+1) fragments
          const float h0 = bf_round(s[nt][0]), h1 = bf_round(s[nt][1]);
          const float h2 = bf_round(s[nt][2]), h3 = bf_round(s[nt][3]);
          ph_[nt][0] = movm_t(pack_bf2(h0, h1));
          ph_[nt][1] = movm_t(pack_bf2(h2, h3));
          pl_[nt][0] = movm_t(pack_bf2(s[nt][0] - h0, s[nt][1] - h1));
          pl_[nt][1] = movm_t(pack_bf2(s[nt][2] - h2, s[nt][3] - h3));
        }
        // ---- O^T += V^T P^T (the lo plane accumulates into its own registers: no serial chain)
#pragma unroll
        for (int dt = 0; dt < DT; ++dt) {
          uint32_t a[4];
          ldsm_x4_t(vb + kvoff<HD>((lane & 7) + ((lane >> 4) & 1) * 8, 2 * dt + ((lane >> 3) & 1), ph.tok0), a);
#pragma unroll
          for (int nt = 0; nt < NQT; ++nt) {
            mma16816(o + (nt * DT + dt) * 4, a, ph_[nt][0], ph_[nt][1]);
            if constexpr (NQT == 1)
              mma16816(olo + (nt * DT + dt) * 4, a, pl_[nt][0], pl_[nt][1]);
            else
              mma16816(o + (nt * DT + dt) * 4, a, pl_[nt][0], pl_[nt][1]);
          }
        }
        ++consumed;
        __syncwarp();
        try_issue();
        if (more) {
#pragma unroll
          for (int nt = 0; nt < NQT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) s[nt][e] = s_next[nt][e];
        }
      }

      if constexpr (NQT == 1) {
#pragma unroll
        for (int i = 0; i < NR; ++i) o[i] += olo[i];
      }
      if (stamp) w.st[8 * blockIdx.x + 4] = ptx::globaltimer();
      // ---- piece epilogue: column sums, then the output (single piece) or a split-KV partial
#pragma unroll
      for (int nt = 0; nt < NQT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          float l = lsum[nt][e];
          l += __shfl_xor_sync(kFull, l, 4);
          l += __shfl_xor_sync(kFull, l, 8);
          l += __shfl_xor_sync(kFull, l, 16);
          lsum[nt][e] = l;
        }
      const int pidx = pb + k;
      const bool single = ph.npieces == 1;
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        const int e = i & 3, dt = (i >> 2) % DT, nt = (i >> 2) / DT;
        const int qi = 8 * nt + 2 * cq + (e & 1);
        const int dim = 16 * dt + gq + (e >> 1) * 8;
        if (qi >= ph.qlen) continue;
        if (single) {
          out[static_cast<size_t>(ph.qs + qi) * D + head * HD + dim] = __float2bfloat16_rn(o[i] / lsum[nt][e & 1]);
        } else {
          const size_t pi = (static_cast<size_t>(pidx) * H + head) * QP + qi;
          w.part_o[pi * HD + dim] = o[i];
          if (dt == 0 && gq == 0 && e < 2) w.part_m[pi] = mrun[nt][e], w.part_l[pi] = lsum[nt][e];
        }
      }
      if (single) continue;
      // ---- arrival: the warp completing the last piece of (request, head) merges them
      __syncwarp();
      int last = 0;
      if (lane == 0) {
        int* cnt = w.counter + static_cast<size_t>(ph.req) * H + head;
        asm volatile("fence.acq_rel.gpu;" ::: "memory");  // release this warp's partial (cumulative via syncwarp)
        last = atomicAdd(cnt, 1) == ph.npieces - 1;
        if (last) {
          asm volatile("fence.acq_rel.gpu;" ::: "memory");  // acquire the other pieces' partials
          *cnt = 0;  // re-armed for the next launch
        }
      }
      last = __shfl_sync(kFull, last, 0);
      if (stamp) w.st[8 * blockIdx.x + 5] = ptx::globaltimer();
      if (!last) continue;
      if (stamp) w.st[8 * blockIdx.x + 6] = ptx::globaltimer();
      // ---- shared-max merge of the request's pieces in token order (attention.cpp:128-157)
      merge_pieces<HD, QP, QP == 8>(m, w, ph, head, H, D, out, lane);
    }
  }
  if (stamp) w.st[8 * blockIdx.x + 7] = ptx::globaltimer();
  ptx::grid_dep_launch();
}

// Warp-specialised verify attention (<= 8 queries per request): one 2-warp CTA per
// (pack row, chunk, head) item. In attn_kernel one warp walks the item's whole tile chain,
// and per 16-key tile that chain is long (S^T = K Q^T, online softmax, movmatrix,
// O^T += V^T P^T): the warp is latency-bound at ~7 resident warps per SM. Here the chain
// is split in two stages that run concurrently on consecutive tiles:
//   warp 0 (scores): K ring, S^T = K Q^T, mask + online softmax (max, sum), P^T fragments
//                    (bf16 hi + lo) + per-query rescale factors -> a double-buffered hand-off;
//   warp 1 (values): V ring, rescales O^T, O^T += V^T P^T, the piece epilogue (output or
//                    split-KV partial) and the last-arriver shared-max merge.
// Each warp issues its own ring (K halves / V halves of the pre-swizzled 16-key tiles),
// so no ring slot waits on the other warp. Same arithmetic as attn_kernel<HD, 1>.
template <int HD>
struct WsCfg {
  static constexpr int kStages = HD == 128 ? 3 : 4;
  static constexpr uint32_t kHalf = 16 * HD * 2;  // K or V of one 16-key tile
  static constexpr uint32_t kRing = 2 * kStages * kHalf;
  static constexpr int kHand = 2 * 32 * 8;        // 2 buffers x 32 lanes x {ph0, ph1, pl0, pl1, corr0, corr1, -, -}
  static constexpr int kPend = 2 * 32 * 4;        // 2 buffers x 32 lanes x {lsum0, lsum1, m0, m1}
  static constexpr size_t kTotal = 1024 + kRing + kMaxPieces * 64 + (kHand + kPend) * 4 + (2 * kStages + 4) * 8;
};

__device__ __forceinline__ void bar_pair(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

template <int HD>
__global__ void __launch_bounds__(64) attn_ws_kernel(FwdMeta m, AttnGeom g, const float* __restrict__ q, AttnWork w,
                                                     bf16* __restrict__ out, int n_items) {
  using WC = WsCfg<HD>;
  constexpr int S = WC::kStages, DT = HD / 16, NR = DT * 4, QP = 8;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int gq = lane >> 2, cq = lane & 3;
  uint8_t* ring = smem + static_cast<size_t>(warp) * S * WC::kHalf;  // warp 0: K ring, warp 1: V ring
  Piece* pcs = reinterpret_cast<Piece*>(smem + WC::kRing);
  float* hand = reinterpret_cast<float*>(smem + WC::kRing + kMaxPieces * 64);
  float* pend = hand + WC::kHand;
  uint64_t* bars = reinterpret_cast<uint64_t*>(pend + WC::kPend);
  uint64_t* full = bars + warp * S;       // this warp's ring
  uint64_t* h_full = bars + 2 * S;        // [2] P hand-off written (32 arrivals)
  uint64_t* h_empty = bars + 2 * S + 2;   // [2] P hand-off read (32 arrivals)
  const int H = g.n_heads, D = H * HD;
  const float sl2 = g.scale * kLog2e;
  const int item = blockIdx.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2 * S; ++s) ptx::mbar_init(&bars[s], 1);
    for (int b = 0; b < 2; ++b) ptx::mbar_init(&h_full[b], 32), ptx::mbar_init(&h_empty[b], 32);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  bool dep_done = false;
  if (!w.early) ptx::grid_dep_wait(), dep_done = true;
  if (item >= n_items * H) return;
  const int head = item % H, rc = item / H;
  const int p_lo = m.item_ptr[rc], p_hi = m.item_ptr[rc + 1];
  const uint64_t pol = ptx::policy_evict_first();
  const int kv_base = (g.layer * g.slots) * H;
  const bf16* cache = warp == 0 ? g.k_cache : g.v_cache;

  int issued = 0, consumed = 0;  // this warp's ring
  int handed = 0;                // P hand-offs produced (warp 0) / consumed (warp 1)
  int piece_no = 0;
  for (int pb = p_lo; pb < p_hi; pb += kMaxPieces) {
    const int np = min(p_hi - pb, kMaxPieces);
    bar_pair(2);  // the previous pass is done with pcs
    for (int k = threadIdx.x; k < np; k += 64) {
      const int4* src = reinterpret_cast<const int4*>(m.pieces + 16 * (pb + k));
      int4* dst = reinterpret_cast<int4*>(pcs + k);
      dst[0] = src[0], dst[1] = src[1], dst[2] = src[2];
    }
    bar_pair(2);
    int ik = 0, it = 0;
    auto try_issue = [&]() {
      while (issued - consumed < S && ik < np) {
        const Piece& ph = pcs[ik];
        if (it * 16 >= ph.len) {
          ++ik, it = 0;
          continue;
        }
        if (!dep_done && ph.tok0 + it * 16 + 16 > ph.kvlen - ph.qlen) break;
        if (lane == 0) {
          const int st = issued % S;
          const size_t r0 = (static_cast<size_t>(kv_base + ph.slot * H + head) * g.ctx) + ph.tok0 + it * 16;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          ptx::mbar_arrive_expect_tx(&full[st], WC::kHalf);
          ptx::bulk_load(ring + st * WC::kHalf, cache + r0 * HD, WC::kHalf, &full[st], pol);
        }
        ++issued;
        ++it;
      }
    };
    try_issue();
    if (!dep_done) {
      ptx::grid_dep_wait();
      dep_done = true;
      try_issue();
    }
    if (pb == p_lo) ptx::grid_dep_launch();

    for (int k = 0; k < np; ++k) {
      const Piece ph = pcs[k];
      const int ntile = (ph.len + 15) / 16;
      const int kend = ph.tok0 + ph.len;
      const int qbase = ph.kvlen - ph.qlen;
      if (warp == 0) {
        // ================================================================ scores warp
        uint32_t qh[DT][2], ql[DT][2];
        {
          const bool ok = gq < ph.qlen;
          const float* qr = q + static_cast<size_t>(ph.qs + (ok ? gq : 0)) * D + head * HD + 2 * cq;
#pragma unroll
          for (int kt = 0; kt < DT; ++kt)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const float2 v =
                  ok ? __ldg(reinterpret_cast<const float2*>(qr + 16 * kt + 8 * hh)) : make_float2(0.f, 0.f);
              const float x = v.x * sl2, y = v.y * sl2;
              const float hx = bf_round(x), hy = bf_round(y);
              qh[kt][hh] = pack_bf2(hx, hy);
              ql[kt][hh] = pack_bf2(x - hx, y - hy);
            }
        }
        float mrun[2] = {-INFINITY, -INFINITY}, lsum[2] = {0.f, 0.f};
        for (int t = 0; t < ntile; ++t) {
          const int st = consumed % S;
          ptx::mbar_wait(&full[st], static_cast<uint32_t>((consumed / S) & 1));
          const uint32_t kb = ptx::smem_u32(ring + st * WC::kHalf);
          float s[4];
          {
            float sc[4][4];
#pragma unroll
            for (int c = 0; c < 4; ++c) sc[c][0] = sc[c][1] = sc[c][2] = sc[c][3] = 0.f;
#pragma unroll
            for (int kt = 0; kt < DT; ++kt) {
              uint32_t a[4];
              ldsm_x4(kb + kvoff<HD>((lane & 7) + ((lane >> 3) & 1) * 8, 2 * kt + (lane >> 4), ph.tok0), a);
              mma16816(sc[kt & 1], a, qh[kt][0], qh[kt][1]);
              mma16816(sc[2 + (kt & 1)], a, ql[kt][0], ql[kt][1]);
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) s[e] = (sc[0][e] + sc[1][e]) + (sc[2][e] + sc[3][e]);
          }
          ++consumed;
          __syncwarp();
          try_issue();  // the K slot is free as soon as the scores are in registers
          const int key0 = ph.tok0 + t * 16 + gq;
          float corr[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int qpos = qbase + 2 * cq + e;
            const bool v0 = key0 < kend && (key0 <= qpos || !g.causal);
            const bool v1 = key0 + 8 < kend && (key0 + 8 <= qpos || !g.causal);
            s[e] = v0 ? s[e] : -INFINITY;
            s[2 + e] = v1 ? s[2 + e] : -INFINITY;
            float mx = fmaxf(s[e], s[2 + e]);
            mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 4));
            mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 8));
            mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 16));
            const float mnew = fmaxf(mrun[e], mx);
            corr[e] = mnew == -INFINITY ? 1.f : exp2f(mrun[e] - mnew);
            const float p0 = mnew == -INFINITY ? 0.f : exp2f(s[e] - mnew);
            const float p1 = mnew == -INFINITY ? 0.f : exp2f(s[2 + e] - mnew);
            s[e] = p0;
            s[2 + e] = p1;
            lsum[e] = lsum[e] * corr[e] + (p0 + p1);
            mrun[e] = mnew;
          }
          const float h0 = bf_round(s[0]), h1 = bf_round(s[1]), h2 = bf_round(s[2]), h3 = bf_round(s[3]);
          const uint32_t ph0 = movm_t(pack_bf2(h0, h1)), ph1 = movm_t(pack_bf2(h2, h3));
          const uint32_t pl0 = movm_t(pack_bf2(s[0] - h0, s[1] - h1)), pl1 = movm_t(pack_bf2(s[2] - h2, s[3] - h3));
          const int hb = handed & 1;
          if (handed >= 2) ptx::mbar_wait(&h_empty[hb], static_cast<uint32_t>(((handed >> 1) - 1) & 1));
          float4* slot = reinterpret_cast<float4*>(hand + (hb * 32 + lane) * 8);
          slot[0] = make_float4(__uint_as_float(ph0), __uint_as_float(ph1), __uint_as_float(pl0), __uint_as_float(pl1));
          slot[1] = make_float4(corr[0], corr[1], 0.f, 0.f);
          ptx::mbar_arrive(&h_full[hb]);
          ++handed;
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          float l = lsum[e];
          l += __shfl_xor_sync(kFull, l, 4);
          l += __shfl_xor_sync(kFull, l, 8);
          l += __shfl_xor_sync(kFull, l, 16);
          lsum[e] = l;
        }
        reinterpret_cast<float4*>(pend)[(piece_no & 1) * 32 + lane] = make_float4(lsum[0], lsum[1], mrun[0], mrun[1]);
        bar_pair(1);  // piece statistics visible to the values warp
      } else {
        // ================================================================ values warp
        float o[NR], olo[NR];
#pragma unroll
        for (int i = 0; i < NR; ++i) o[i] = olo[i] = 0.f;
        for (int t = 0; t < ntile; ++t) {
          const int st = consumed % S;
          const int hb = handed & 1;
          ptx::mbar_wait(&h_full[hb], static_cast<uint32_t>((handed >> 1) & 1));
          const float4* slot = reinterpret_cast<const float4*>(hand + (hb * 32 + lane) * 8);
          const float4 pv = slot[0], cr = slot[1];
          ptx::mbar_arrive(&h_empty[hb]);
          ++handed;
          const uint32_t ph0 = __float_as_uint(pv.x), ph1 = __float_as_uint(pv.y);
          const uint32_t pl0 = __float_as_uint(pv.z), pl1 = __float_as_uint(pv.w);
#pragma unroll
          for (int dt = 0; dt < DT; ++dt) {
            float* oo = o + dt * 4;
            oo[0] *= cr.x, oo[1] *= cr.y, oo[2] *= cr.x, oo[3] *= cr.y;
            float* ol = olo + dt * 4;
            ol[0] *= cr.x, ol[1] *= cr.y, ol[2] *= cr.x, ol[3] *= cr.y;
          }
          ptx::mbar_wait(&full[st], static_cast<uint32_t>((consumed / S) & 1));
          const uint32_t vb = ptx::smem_u32(ring + st * WC::kHalf);
#pragma unroll
          for (int dt = 0; dt < DT; ++dt) {
            uint32_t a[4];
            ldsm_x4_t(vb + kvoff<HD>((lane & 7) + ((lane >> 4) & 1) * 8, 2 * dt + ((lane >> 3) & 1), ph.tok0), a);
            mma16816(o + dt * 4, a, ph0, ph1);
            mma16816(olo + dt * 4, a, pl0, pl1);
          }
          ++consumed;
          __syncwarp();
          try_issue();
        }
#pragma unroll
        for (int i = 0; i < NR; ++i) o[i] += olo[i];
        bar_pair(1);  // the scores warp's piece statistics
        const float4 ps = reinterpret_cast<const float4*>(pend)[(piece_no & 1) * 32 + lane];
        const float lsum[2] = {ps.x, ps.y}, mrun[2] = {ps.z, ps.w};
        // ---- piece epilogue: the output (single piece) or a split-KV partial
        const int pidx = pb + k;
        const bool single = ph.npieces == 1;
#pragma unroll
        for (int i = 0; i < NR; ++i) {
          const int e = i & 3, dt = i >> 2;
          const int qi = 2 * cq + (e & 1);
          const int dim = 16 * dt + gq + (e >> 1) * 8;
          if (qi >= ph.qlen) continue;
          if (single) {
            out[static_cast<size_t>(ph.qs + qi) * D + head * HD + dim] = __float2bfloat16_rn(o[i] / lsum[e & 1]);
          } else {
            const size_t pi = (static_cast<size_t>(pidx) * H + head) * QP + qi;
            w.part_o[pi * HD + dim] = o[i];
            if (dt == 0 && gq == 0 && e < 2) w.part_m[pi] = mrun[e], w.part_l[pi] = lsum[e];
          }
        }
        if (!single) {
          // ---- arrival: the warp completing the last piece of (request, head) merges them
          __syncwarp();
          int last = 0;
          if (lane == 0) {
            int* cnt = w.counter + static_cast<size_t>(ph.req) * H + head;
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            last = atomicAdd(cnt, 1) == ph.npieces - 1;
            if (last) {
              asm volatile("fence.acq_rel.gpu;" ::: "memory");
              *cnt = 0;  // re-armed for the next launch
            }
          }
          last = __shfl_sync(kFull, last, 0);
          if (last) merge_pieces<HD, QP, true>(m, w, ph, head, H, D, out, lane);
        }
      }
      ++piece_no;
    }
  }
  ptx::grid_dep_launch();
}

// Multi-query verify attention (9..8*NQW queries per request: ragged / long windows): one CTA
// per (pack row, chunk, head) item, NQW consumer warps + one producer warp sharing ONE K/V
// ring. Consumer warp w owns queries 8w..8w+7 of every piece (attn_kernel<HD, 1>'s per-warp
// arithmetic: hi / lo Q and P planes, separate lo accumulator chain, scores of tile t + 1
// issued before tile t's softmax), so every 16-key tile is read from DRAM once for all of a
// request's queries, a warp whose query tile is empty for the piece (qlen <= 8w) only passes
// the tile on, and each warp's register budget is the one-tile kernel's (attn_kernel<128, 3>
// carried 3 tiles per warp and spilled). The producer's lane 0 streams the item's tiles
// (1-D bulk copies of the pre-swizzled cache rows) and recycles a slot once every consumer
// warp released it (empty barrier, NQW arrivals). Split-KV pieces: the consumer warps meet at
// a named barrier, warp 0 takes the arrival ticket and, last, merges (merge_pieces).
template <int HD, int NQW, int ST>
struct MqCfg {
  static constexpr int kStages = ST;
  static constexpr uint32_t kHalf = 16 * HD * 2;
  static constexpr uint32_t kStage = 2 * kHalf;
  static constexpr int kDT = HD / 16;
  static constexpr int kNR = kDT * 4;
  static constexpr int kQP = 8 * NQW;
  static constexpr size_t kTotal = 1024 + kStages * kStage + 2 * kStages * 8;
};

template <int HD, int NQW, int ST>
__global__ void __launch_bounds__(32 * (NQW + 1)) attn_mq_kernel(FwdMeta m, AttnGeom g, const float* __restrict__ q,
                                                                 AttnWork w, bf16* __restrict__ out) {
  using C = MqCfg<HD, NQW, ST>;
  constexpr int S = C::kStages, DT = C::kDT, NR = C::kNR, QP = C::kQP;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * C::kStage);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int gq = lane >> 2, cq = lane & 3;
  const int H = g.n_heads, D = H * HD;
  const float sl2 = g.scale * kLog2e;
  const int head = blockIdx.x % H, rc = blockIdx.x / H;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) ptx::mbar_init(&full[s], 1), ptx::mbar_init(&empty[s], NQW);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const bool stamp = w.st != nullptr && threadIdx.x == 0;
  if (stamp) w.st[8 * blockIdx.x] = ptx::globaltimer();
  // w.early: the work list and the KV rows older than the queries are complete before this
  // grid starts (attn_kernel), so the producer issues those tiles before the dependency wait
  const int p_lo = m.item_ptr[rc], p_hi = m.item_ptr[rc + 1];
  const Piece* pieces = reinterpret_cast<const Piece*>(m.pieces);
  if (warp == NQW) {  // ---- producer
    if (lane == 0) {
      bool dep = !w.early;
      if (dep) ptx::grid_dep_wait();
      const uint64_t pol = ptx::policy_evict_first();
      const size_t kv_base = static_cast<size_t>(g.layer * g.slots) * H;
      int issued = 0;
      for (int p = p_lo; p < p_hi; ++p) {
        const int slot = pieces[p].slot, tok0 = pieces[p].tok0, len = pieces[p].len;
        const int fresh = pieces[p].kvlen - pieces[p].qlen;  // first key written by this forward
        const size_t row0 = ((kv_base + static_cast<size_t>(slot) * H + head) * g.ctx) + tok0;
        for (int t = 0; t * 16 < len; ++t, ++issued) {
          if (!dep && tok0 + t * 16 + 16 > fresh) ptx::grid_dep_wait(), dep = true;
          const int st = issued % S;
          if (issued >= S) ptx::mbar_wait(&empty[st], static_cast<uint32_t>(((issued / S) - 1) & 1));
          uint8_t* dst = ring + st * C::kStage;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          ptx::mbar_arrive_expect_tx(&full[st], C::kStage);
          ptx::bulk_load(dst, g.k_cache + (row0 + t * 16) * HD, C::kHalf, &full[st], pol);
          ptx::bulk_load(dst + C::kHalf, g.v_cache + (row0 + t * 16) * HD, C::kHalf, &full[st], pol);
        }
      }
    }
    ptx::grid_dep_launch();
    return;
  }
  // ---- consumers: queries 8 * warp .. 8 * warp + 7 of every piece
  ptx::grid_dep_wait();  // q (and this forward's new keys) come from the QKV epilogue
  ptx::grid_dep_launch();
  int consumed = 0;
  for (int p = p_lo; p < p_hi; ++p) {
    const Piece ph = pieces[p];
    const int ntile = (ph.len + 15) / 16;
    if (8 * warp >= ph.qlen) {  // no query of this warp in the piece: pass its tiles on
      for (int t = 0; t < ntile; ++t, ++consumed) {
        ptx::mbar_wait(&full[consumed % S], static_cast<uint32_t>((consumed / S) & 1));
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&empty[consumed % S]);
      }
    } else {
      uint32_t qh[DT][2], ql[DT][2];
      {
        const int qi = 8 * warp + gq;
        const bool ok = qi < ph.qlen;
        const float* qr = q + static_cast<size_t>(ph.qs + (ok ? qi : 0)) * D + head * HD + 2 * cq;
#pragma unroll
        for (int kt = 0; kt < DT; ++kt)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const float2 v = ok ? __ldg(reinterpret_cast<const float2*>(qr + 16 * kt + 8 * hh)) : make_float2(0.f, 0.f);
            const float x = v.x * sl2, y = v.y * sl2;
            const float hx = bf_round(x), hy = bf_round(y);
            qh[kt][hh] = pack_bf2(hx, hy);
            ql[kt][hh] = pack_bf2(x - hx, y - hy);
          }
      }
      float o[NR], olo[NR];
#pragma unroll
      for (int i = 0; i < NR; ++i) o[i] = 0.f, olo[i] = 0.f;
      float mrun[2] = {-INFINITY, -INFINITY}, lsum[2] = {0.f, 0.f};
      const int qbase = ph.kvlen - ph.qlen;
      auto scores = [&](int stg, float (&sv)[4]) {
        const uint32_t kb = ptx::smem_u32(ring + stg * C::kStage);
        float sc[4][4];
#pragma unroll
        for (int c = 0; c < 4; ++c) sc[c][0] = sc[c][1] = sc[c][2] = sc[c][3] = 0.f;
#pragma unroll
        for (int kt = 0; kt < DT; ++kt) {
          uint32_t a[4];
          ldsm_x4(kb + kvoff<HD>((lane & 7) + ((lane >> 3) & 1) * 8, 2 * kt + (lane >> 4), ph.tok0), a);
          mma16816(sc[kt & 1], a, qh[kt][0], qh[kt][1]);
          mma16816(sc[2 + (kt & 1)], a, ql[kt][0], ql[kt][1]);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) sv[e] = (sc[0][e] + sc[1][e]) + (sc[2][e] + sc[3][e]);
      };
      float s[4];
      ptx::mbar_wait(&full[consumed % S], static_cast<uint32_t>((consumed / S) & 1));
      scores(consumed % S, s);
      for (int t = 0; t < ntile; ++t, ++consumed) {
        const int st = consumed % S;
        const bool more = t + 1 < ntile;
        float s_next[4];
        if (more) {
          const int st1 = (consumed + 1) % S;
          ptx::mbar_wait(&full[st1], static_cast<uint32_t>(((consumed + 1) / S) & 1));
          scores(st1, s_next);
        }
        const uint32_t vb = ptx::smem_u32(ring + st * C::kStage) + C::kHalf;
        const int key0 = ph.tok0 + t * 16 + gq;
        const int kend = ph.tok0 + ph.len;
        float corr[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int qpos = qbase + 8 * warp + 2 * cq + e;
          const bool v0 = key0 < kend && (key0 <= qpos || !g.causal);
          const bool v1 = key0 + 8 < kend && (key0 + 8 <= qpos || !g.causal);
          s[e] = v0 ? s[e] : -INFINITY;
          s[2 + e] = v1 ? s[2 + e] : -INFINITY;
          float mx = fmaxf(s[e], s[2 + e]);
          mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 4));
          mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 8));
          mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 16));
          const float mnew = fmaxf(mrun[e], mx);
          corr[e] = mnew == -INFINITY ? 1.f : exp2f(mrun[e] - mnew);
          const float p0 = mnew == -INFINITY ? 0.f : exp2f(s[e] - mnew);
          const float p1 = mnew == -INFINITY ? 0.f : exp2f(s[2 + e] - mnew);
          s[e] = p0;
          s[2 + e] = p1;
          lsum[e] = lsum[e] * corr[e] + (p0 + p1);
          mrun[e] = mnew;
        }
#pragma unroll
        for (int dt = 0; dt < DT; ++dt) {
          float* oo = o + dt * 4;
          float* ol = olo + dt * 4;
          oo[0] *= corr[0], oo[1] *= corr[1], oo[2] *= corr[0], oo[3] *= corr[1];
          ol[0] *= corr[0], ol[1] *= corr[1], ol[2] *= corr[0], ol[3] *= corr[1];
        }
        const float h0 = bf_round(s[0]), h1 = bf_round(s[1]), h2 = bf_round(s[2]), h3 = bf_round(s[3]);
        const uint32_t ph0 = movm_t(pack_bf2(h0, h1)), ph1 = movm_t(pack_bf2(h2, h3));
        const uint32_t pl0 = movm_t(pack_bf2(s[0] - h0, s[1] - h1)), pl1 = movm_t(pack_bf2(s[2] - h2, s[3] - h3));
#pragma unroll
        for (int dt = 0; dt < DT; ++dt) {
          uint32_t a[4];
          ldsm_x4_t(vb + kvoff<HD>((lane & 7) + ((lane >> 4) & 1) * 8, 2 * dt + ((lane >> 3) & 1), ph.tok0), a);
          mma16816(o + dt * 4, a, ph0, ph1);
          mma16816(olo + dt * 4, a, pl0, pl1);
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&empty[st]);
        if (more) {
#pragma unroll
          for (int e = 0; e < 4; ++e) s[e] = s_next[e];
        }
      }
#pragma unroll
      for (int i = 0; i < NR; ++i) o[i] += olo[i];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        float l = lsum[e];
        l += __shfl_xor_sync(kFull, l, 4);
        l += __shfl_xor_sync(kFull, l, 8);
        l += __shfl_xor_sync(kFull, l, 16);
        lsum[e] = l;
      }
      const bool single = ph.npieces == 1;
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        const int e = i & 3, dt = i >> 2;
        const int qi = 8 * warp + 2 * cq + (e & 1);
        const int dim = 16 * dt + gq + (e >> 1) * 8;
        if (qi >= ph.qlen) continue;
        if (single) {
          out[static_cast<size_t>(ph.qs + qi) * D + head * HD + dim] = __float2bfloat16_rn(o[i] / lsum[e & 1]);
        } else {
          const size_t pi = (static_cast<size_t>(p) * H + head) * QP + qi;
          w.part_o[pi * HD + dim] = o[i];
          if (dt == 0 && gq == 0 && e < 2) w.part_m[pi] = mrun[e], w.part_l[pi] = lsum[e];
        }
      }
    }
    if (ph.npieces == 1) continue;
    // ---- every consumer warp's partial of this piece is written: arrival, last merges
    asm volatile("bar.sync 1, %0;" ::"r"(32 * NQW) : "memory");
    if (warp != 0) continue;
    int last = 0;
    if (lane == 0) {
      int* cnt = w.counter + static_cast<size_t>(ph.req) * H + head;
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      last = atomicAdd(cnt, 1) == ph.npieces - 1;
      if (last) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        *cnt = 0;
      }
    }
    last = __shfl_sync(kFull, last, 0);
    if (last) merge_pieces<HD, QP, false>(m, w, ph, head, H, D, out, lane);
  }
  if (stamp) w.st[8 * blockIdx.x + 7] = ptx::globaltimer();
}

// Few-query (draft step) variant: one CTA per (pack row, chunk, head) item whose four
// warps take the item's 16-key tiles round robin, so the longest chain is a quarter of
// a chunk (one ring's worth: a single DRAM round trip) instead of a whole chunk; the
// warps' partials of each piece are merged in shared memory (fixed warp order), and
// pieces of multi-piece requests go through the same global last-arriver merge as
// attn_kernel. NQT = 1 (<= 8 queries per request).
template <int HD, int ST>
struct DecCfg {
  using C = Cfg<HD, 1, kNW, ST>;
  static constexpr int kQ = kDecodeQ;                // queries per request (<= 2)
  static constexpr int kMergeFloats = kQ * (2 + HD);  // per slot: m[kQ], l[kQ], o[kQ][HD]
  static constexpr int kCluster = 2;                 // CTAs per item (tiles round robin over 2 x 4 warps)
  static constexpr size_t kTotal = 1024 + C::kRing + kMaxPieces * 64 + kNW * C::kStages * 8 +
                                   (kNW + kCluster) * kMergeFloats * 4;  // warp slots + cluster receive slots
};

template <int HD, int ST>
__global__ void __launch_bounds__(kThreads) attn_decode_kernel(FwdMeta m, AttnGeom g, const float* __restrict__ q,
                                                               AttnWork w, bf16* __restrict__ out, int n_items) {
  using DC = DecCfg<HD, ST>;
  using C = typename DC::C;
  constexpr int CS = DC::kCluster;
  constexpr int S = C::kStages, DT = C::kDT, NR = C::kNR, QP = C::kQP;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int gq = lane >> 2, cq = lane & 3;
  uint8_t* ring = smem + static_cast<size_t>(warp) * S * C::kStage;
  Piece* pcs = reinterpret_cast<Piece*>(smem + C::kRing);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::kRing + kMaxPieces * 64) + warp * S;
  float* mrg = reinterpret_cast<float*>(smem + C::kRing + kMaxPieces * 64 + kNW * S * 8);
  constexpr int kQ = DC::kQ;
  float* my_m = mrg + warp * DC::kMergeFloats;  // [kQ]
  float* my_l = my_m + kQ;                       // [kQ]
  float* my_o = my_m + 2 * kQ;                   // [kQ][HD]
  float* rcv = mrg + kNW * DC::kMergeFloats;     // [CS] CTA partials, filled over DSMEM (rank 0 reads)
  const int H = g.n_heads, D = H * HD;
  const float sl2 = g.scale * kLog2e;
  const int item = blockIdx.x / CS;  // (pack row, chunk) x head; a cluster of CS CTAs per item
  const int crank = static_cast<int>(ptx::cluster_ctarank());
  const int vwarp = crank * kNW + warp, vwarps = CS * kNW;  // tiles round robin over the cluster's warps
  ptx::cluster_arrive_relaxed();  // (waited before the first remote store: every CTA has started)
  if (lane == 0) {
    for (int s = 0; s < S; ++s) ptx::mbar_init(&bar[s], 1);
    ptx::fence_mbar_init();
  }
  __syncwarp();
  const bool stamp = w.st != nullptr && threadIdx.x == 0;
  if (stamp) w.st[8 * blockIdx.x] = ptx::globaltimer();
  bool dep_done = false;
  if (!w.early) ptx::grid_dep_wait(), dep_done = true;
  const int head = item % H, rc = item / H;
  const int p_lo = m.item_ptr[rc], p_hi = m.item_ptr[rc + 1];
  const uint64_t pol = ptx::policy_evict_first();
  const int kv_base = (g.layer * g.slots) * H;

  int issued = 0, consumed = 0;
  for (int pb = p_lo; pb < p_hi; pb += kMaxPieces) {
    const int np = min(p_hi - pb, kMaxPieces);
    __syncthreads();  // previous pass done with pcs
    for (int k = threadIdx.x; k < np; k += kThreads) {
      const int4* src = reinterpret_cast<const int4*>(m.pieces + 16 * (pb + k));
      int4* dst = reinterpret_cast<int4*>(pcs + k);
      dst[0] = src[0], dst[1] = src[1], dst[2] = src[2];
    }
    __syncthreads();
    // this warp's tiles: every vwarps-th tile of the pass's tile sequence (pieces in order)
    int ik = 0, it = vwarp;
    auto norm_pos = [&]() {
      while (ik < np && it * 16 >= pcs[ik].len) it -= (pcs[ik].len + 15) / 16, ++ik;
    };
    norm_pos();
    auto try_issue = [&]() {
      while (issued - consumed < S && ik < np) {
        const Piece& ph = pcs[ik];
        if (!dep_done && ph.tok0 + it * 16 + 16 > ph.kvlen - ph.qlen) break;
        if (lane == 0) {
          const int st = issued % S;
          uint8_t* dst = ring + st * C::kStage;
          const size_t r0 = (static_cast<size_t>(kv_base + ph.slot * H + head) * g.ctx) + ph.tok0 + it * 16;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          ptx::mbar_arrive_expect_tx(&bar[st], C::kStage);
          ptx::bulk_load(dst, g.k_cache + r0 * HD, C::kHalf, &bar[st], pol);
          ptx::bulk_load(dst + C::kHalf, g.v_cache + r0 * HD, C::kHalf, &bar[st], pol);
        }
        ++issued;
        it += vwarps;
        norm_pos();
      }
    };
    try_issue();
    if (!dep_done) {
      ptx::grid_dep_wait();
      ptx::grid_dep_launch();
      dep_done = true;
      if (stamp) w.st[8 * blockIdx.x + 1] = ptx::globaltimer();
      try_issue();
    }

    int tile_base = 0;  // first tile index of piece k in the pass's sequence
    for (int k = 0; k < np; ++k) {
      const Piece ph = pcs[k];
      const int n_tiles = (ph.len + 15) / 16;
      uint32_t qh[DT][2], ql[DT][2];
      {
        const int qi = gq;
        const bool ok = qi < ph.qlen;
        const float* qr = q + static_cast<size_t>(ph.qs + (ok ? qi : 0)) * D + head * HD + 2 * cq;
#pragma unroll
        for (int kt = 0; kt < DT; ++kt)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const float2 v =
                ok ? __ldg(reinterpret_cast<const float2*>(qr + 16 * kt + 8 * hh)) : make_float2(0.f, 0.f);
            const float x = v.x * sl2, y = v.y * sl2;
            const float hx = bf_round(x), hy = bf_round(y);
            qh[kt][hh] = pack_bf2(hx, hy);
            ql[kt][hh] = pack_bf2(x - hx, y - hy);
          }
      }
      float o[NR], olo[NR];
#pragma unroll
      for (int i = 0; i < NR; ++i) o[i] = olo[i] = 0.f;
      float mrun[2] = {-INFINITY, -INFINITY}, lsum[2] = {0.f, 0.f};
      const int qbase = ph.kvlen - ph.qlen;
      // tiles t of this piece with (tile_base + t) % vwarps == vwarp
      int t = (vwarp - tile_base % vwarps + vwarps) % vwarps;
      for (; t < n_tiles; t += vwarps) {
        const int st = consumed % S;
        ptx::mbar_wait(&bar[st], static_cast<uint32_t>((consumed / S) & 1));
        const uint32_t kb = ptx::smem_u32(ring + st * C::kStage);
        const uint32_t vb = kb + C::kHalf;
        float s[4];
        {
          float sc[4][4];
#pragma unroll
          for (int c = 0; c < 4; ++c) sc[c][0] = sc[c][1] = sc[c][2] = sc[c][3] = 0.f;
#pragma unroll
          for (int kt = 0; kt < DT; ++kt) {
            uint32_t a[4];
            ldsm_x4(kb + kvoff<HD>((lane & 7) + ((lane >> 3) & 1) * 8, 2 * kt + (lane >> 4), ph.tok0), a);
            mma16816(sc[kt & 1], a, qh[kt][0], qh[kt][1]);
            mma16816(sc[2 + (kt & 1)], a, ql[kt][0], ql[kt][1]);
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) s[e] = (sc[0][e] + sc[1][e]) + (sc[2][e] + sc[3][e]);
        }
        const int key0 = ph.tok0 + t * 16 + gq;
        const int kend = ph.tok0 + ph.len;
        float corr[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int qpos = qbase + 2 * cq + e;
          const bool v0 = key0 < kend && (key0 <= qpos || !g.causal);
          const bool v1 = key0 + 8 < kend && (key0 + 8 <= qpos || !g.causal);
          s[e] = v0 ? s[e] : -INFINITY;
          s[2 + e] = v1 ? s[2 + e] : -INFINITY;
          float mx = fmaxf(s[e], s[2 + e]);
          mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 4));
          mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 8));
          mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 16));
          const float mnew = fmaxf(mrun[e], mx);
          corr[e] = mnew == -INFINITY ? 1.f : exp2f(mrun[e] - mnew);
          const float p0 = mnew == -INFINITY ? 0.f : exp2f(s[e] - mnew);
          const float p1 = mnew == -INFINITY ? 0.f : exp2f(s[2 + e] - mnew);
          s[e] = p0;
          s[2 + e] = p1;
          lsum[e] = lsum[e] * corr[e] + (p0 + p1);
          mrun[e] = mnew;
        }
#pragma unroll
        for (int dt = 0; dt < DT; ++dt) {
          float* oo = o + dt * 4;
          oo[0] *= corr[0], oo[1] *= corr[1], oo[2] *= corr[0], oo[3] *= corr[1];
          float* ol = olo + dt * 4;
          ol[0] *= corr[0], ol[1] *= corr[1], ol[2] *= corr[0], ol[3] *= corr[1];
        }
        const float h0 = bf_round(s[0]), h1 = bf_round(s[1]), h2 = bf_round(s[2]), h3 = bf_round(s[3]);
        const uint32_t ph0 = movm_t(pack_bf2(h0, h1)), ph1 = movm_t(pack_bf2(h2, h3));
        const uint32_t pl0 = movm_t(pack_bf2(s[0] - h0, s[1] - h1)), pl1 = movm_t(pack_bf2(s[2] - h2, s[3] - h3));
#pragma unroll
        for (int dt = 0; dt < DT; ++dt) {
          uint32_t a[4];
          ldsm_x4_t(vb + kvoff<HD>((lane & 7) + ((lane >> 4) & 1) * 8, 2 * dt + ((lane >> 3) & 1), ph.tok0), a);
          mma16816(o + dt * 4, a, ph0, ph1);
          mma16816(olo + dt * 4, a, pl0, pl1);
        }
        ++consumed;
        __syncwarp();
        try_issue();
      }
      tile_base += n_tiles;
#pragma unroll
      for (int i = 0; i < NR; ++i) o[i] += olo[i];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        float l = lsum[e];
        l += __shfl_xor_sync(kFull, l, 4);
        l += __shfl_xor_sync(kFull, l, 8);
        l += __shfl_xor_sync(kFull, l, 16);
        lsum[e] = l;
      }
      if (stamp && k == 0) w.st[8 * blockIdx.x + 4] = ptx::globaltimer();
      // ---- this warp's partial of the piece -> shared memory
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        const int e = i & 3, dt = i >> 2;
        const int qi = 2 * cq + (e & 1);
        const int dim = 16 * dt + gq + (e >> 1) * 8;
        if (qi >= kQ) continue;
        my_o[qi * HD + dim] = o[i];
        if (dt == 0 && gq == 0 && e < 2) my_m[qi] = mrun[e], my_l[qi] = lsum[e];
      }
      __syncthreads();
      // ---- fixed-order merge of the four warps' partials into this CTA's partial, stored
      // into receive slot `crank` of the cluster's rank-0 CTA (shared memory over DSMEM)
      if (k == 0 && pb == p_lo) ptx::cluster_wait();  // every CTA of the cluster has started
      const uint32_t slot0 = ptx::mapa(ptx::smem_u32(rcv + crank * DC::kMergeFloats), 0);
      for (int x = threadIdx.x; x < ph.qlen * HD; x += kThreads) {
        const int qi = x / HD, dim = x % HD;
        float M = -INFINITY;
#pragma unroll
        for (int ww = 0; ww < kNW; ++ww) M = fmaxf(M, mrg[ww * DC::kMergeFloats + qi]);
        float L = 0.f, O = 0.f;
#pragma unroll
        for (int ww = 0; ww < kNW; ++ww) {
          const float* wm = mrg + ww * DC::kMergeFloats;
          const float f = wm[qi] == -INFINITY ? 0.f : exp2f(wm[qi] - M);
          L += wm[kQ + qi] * f;
          O += wm[2 * kQ + qi * HD + dim] * f;
        }
        ptx::st_cluster_f32(slot0 + 4u * (2 * kQ + qi * HD + dim), O);
        if (dim == 0) ptx::st_cluster_f32(slot0 + 4u * qi, M), ptx::st_cluster_f32(slot0 + 4u * (kQ + qi), L);
      }
      ptx::cluster_arrive();
      ptx::cluster_wait();  // rank 0 holds every CTA partial of the piece
      const bool single = ph.npieces == 1;
      const int pidx = pb + k;
      if (crank == 0) {
        for (int x = threadIdx.x; x < ph.qlen * HD; x += kThreads) {
          const int qi = x / HD, dim = x % HD;
          float M = -INFINITY;
#pragma unroll
          for (int r = 0; r < CS; ++r) M = fmaxf(M, rcv[r * DC::kMergeFloats + qi]);
          float L = 0.f, O = 0.f;
#pragma unroll
          for (int r = 0; r < CS; ++r) {
            const float* rm = rcv + r * DC::kMergeFloats;
            const float f = rm[qi] == -INFINITY ? 0.f : exp2f(rm[qi] - M);
            L += rm[kQ + qi] * f;
            O += rm[2 * kQ + qi * HD + dim] * f;
          }
          if (single) {
            out[static_cast<size_t>(ph.qs + qi) * D + head * HD + dim] = __float2bfloat16_rn(O / L);
          } else {
            const size_t pi = (static_cast<size_t>(pidx) * H + head) * QP + qi;
            w.part_o[pi * HD + dim] = O;
            if (dim == 0) w.part_m[pi] = M, w.part_l[pi] = L;
          }
        }
      }
      if (pb + k + 1 < p_hi) {  // another piece follows: slots are reused
        ptx::cluster_arrive();
        ptx::cluster_wait();
      } else {
        __syncthreads();  // partial complete before the arrival below
      }
      if (stamp && k == 0) w.st[8 * blockIdx.x + 5] = ptx::globaltimer();
      if (single || crank != 0 || warp != 0) continue;
      // ---- arrival: the CTA completing the last piece of (request, head) merges them
      int last = 0;
      if (lane == 0) {
        int* cnt = w.counter + static_cast<size_t>(ph.req) * H + head;
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        last = atomicAdd(cnt, 1) == ph.npieces - 1;
        if (last) {
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          *cnt = 0;
        }
      }
      last = __shfl_sync(kFull, last, 0);
      if (!last) continue;
      if (stamp) w.st[8 * blockIdx.x + 6] = ptx::globaltimer();
      merge_pieces<HD, QP, QP == 8>(m, w, ph, head, H, D, out, lane);
    }
  }
  if (stamp) w.st[8 * blockIdx.x + 7] = ptx::globaltimer();

}

template <int HD, int ST>
void launch_decode_st(const FwdMeta& m, int n_rows, const AttnGeom& g, const float* q, const AttnWork& w, bf16* out,
                      cudaStream_t s) {
  using DC = DecCfg<HD, ST>;
  ensure_smem_optin(reinterpret_cast<const void*>(attn_decode_kernel<HD, ST>), DC::kTotal);
  const int n_items = n_rows * std::max(1, w.chunks);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_allowed();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.stream = s;
  cudaLaunchAttribute attr2[2];
  attr2[0] = attr[0];
  attr2[1].id = cudaLaunchAttributeClusterDimension;
  attr2[1].val.clusterDim.x = DC::kCluster;
  attr2[1].val.clusterDim.y = 1;
  attr2[1].val.clusterDim.z = 1;
  cfg.attrs = attr2;
  cfg.numAttrs = 2;
  cfg.gridDim = dim3(n_items * g.n_heads * DC::kCluster);  // one cluster per (row, chunk, head)
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = DC::kTotal;
  cudaLaunchKernelEx(&cfg, attn_decode_kernel<HD, ST>, m, g, q, w, out, n_items);
}

// Ring depth of the few-query kernel: a draft-step item is a whole (request, head) over
// 2 x 4 warps, a few 16-key tiles per warp, so a shallow ring keeps the CTA small enough
// for every item of a launch to be resident at once (one wave).
template <int HD>
void launch_decode(const FwdMeta& m, int n_rows, const AttnGeom& g, const float* q, const AttnWork& w, bf16* out,
                   cudaStream_t s) {
  static const int st = [] {
    const char* e = std::getenv("SPIN_ATTN_DEC_STAGES");  // tuning
    return e ? std::atoi(e) : kDecStages;
  }();
  if (st <= 2) return launch_decode_st<HD, 2>(m, n_rows, g, q, w, out, s);
  if (st == 3) return launch_decode_st<HD, 3>(m, n_rows, g, q, w, out, s);
  return launch_decode_st<HD, 4>(m, n_rows, g, q, w, out, s);
}

template <int HD, int NQT>
void launch_t(const CUtensorMap& tm_k, const CUtensorMap& tm_v, const FwdMeta& m, int n_rows, const AttnGeom& g,
              const float* q, const AttnWork& w, bf16* out, cudaStream_t s) {
  using C = Cfg<HD, NQT, kVW>;
  ensure_smem_optin(reinterpret_cast<const void*>(attn_kernel<HD, NQT>), C::kTotal);
  const int n_items = n_rows * std::max(1, w.chunks);
  static const int early = [] {
    const char* e = std::getenv("SPIN_ATTN_EARLY");  // experiments only: 0 disables
    return e ? std::atoi(e) : 1;
  }();
  AttnWork wk = w;
  wk.early = w.early && early;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_allowed();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.stream = s;
  cfg.gridDim = dim3((n_items * g.n_heads + kVW - 1) / kVW);  // one warp per (row, chunk, head)
  cfg.blockDim = dim3(32 * kVW);
  cfg.dynamicSmemBytes = C::kTotal;
  cudaLaunchKernelEx(&cfg, attn_kernel<HD, NQT>, tm_k, tm_v, m, g, q, wk, out, n_items);
}

template <int HD>
void launch_ws(const FwdMeta& m, int n_rows, const AttnGeom& g, const float* q, const AttnWork& w, bf16* out,
               cudaStream_t s) {
  using WC = WsCfg<HD>;
  ensure_smem_optin(reinterpret_cast<const void*>(attn_ws_kernel<HD>), WC::kTotal);
  static const int early = [] {
    const char* e = std::getenv("SPIN_ATTN_EARLY");  // experiments only: 0 disables
    return e ? std::atoi(e) : 1;
  }();
  AttnWork wk = w;
  wk.early = w.early && early;
  const int n_items = n_rows * std::max(1, w.chunks);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_allowed();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.stream = s;
  cfg.gridDim = dim3(n_items * g.n_heads);  // one 2-warp CTA per (row, chunk, head)
  cfg.blockDim = dim3(64);
  cfg.dynamicSmemBytes = WC::kTotal;
  cudaLaunchKernelEx(&cfg, attn_ws_kernel<HD>, m, g, q, wk, out, n_items);
}

template <int HD, int NQW, int ST>
void launch_mq_st(const FwdMeta& m, int n_rows, const AttnGeom& g, const float* q, const AttnWork& w, bf16* out,
                  cudaStream_t s) {
  using MC = MqCfg<HD, NQW, ST>;
  ensure_smem_optin(reinterpret_cast<const void*>(attn_mq_kernel<HD, NQW, ST>), MC::kTotal);
  static const int early = [] {
    const char* e = std::getenv("SPIN_ATTN_EARLY");  // experiments only: 0 disables
    return e ? std::atoi(e) : 1;
  }();
  AttnWork wk = w;
  wk.early = w.early && early;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_allowed();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.stream = s;
  cfg.gridDim = dim3(n_rows * std::max(1, w.chunks) * g.n_heads);  // one CTA per (row, chunk, head)
  cfg.blockDim = dim3(32 * (NQW + 1));
  cfg.dynamicSmemBytes = MC::kTotal;
  cudaLaunchKernelEx(&cfg, attn_mq_kernel<HD, NQW, ST>, m, g, q, wk, out);
}

template <int HD, int NQW>
void launch_mq(const FwdMeta& m, int n_rows, const AttnGeom& g, const float* q, const AttnWork& w, bf16* out,
               cudaStream_t s) {
  static const int st = [] {
    const char* e = std::getenv("SPIN_ATTN_MQ_STAGES");  // tuning
    return e ? std::atoi(e) : 4;
  }();
  if (st <= 4) return launch_mq_st<HD, NQW, 4>(m, n_rows, g, q, w, out, s);
  if (st <= 8) return launch_mq_st<HD, NQW, 8>(m, n_rows, g, q, w, out, s);
  return launch_mq_st<HD, NQW, 12>(m, n_rows, g, q, w, out, s);
}

// attn_mq_kernel serves windows of 9..24 queries; SPIN_ATTN_MQ=0 sends them to
// attn_kernel<HD, 2 / 3> (one warp carrying every query tile; A/B)
bool mq_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("SPIN_ATTN_MQ");
    return e ? std::atoi(e) != 0 : true;
  }();
  return v;
}

template <int HD>
void launch_hd(const CUtensorMap& tm_k, const CUtensorMap& tm_v, const FwdMeta& m, int n_rows, const AttnGeom& g,
               const float* q, const AttnWork& w, bf16* out, cudaStream_t s) {
  static const bool ws = [] {
    // A/B switch, off by default: the warp-specialised kernel measured equal to attn_kernel
    // at config 2 (47.1 vs 46.8 us per layer in situ, round 2)
    const char* e = std::getenv("SPIN_ATTN_WS");
    return e ? std::atoi(e) != 0 : false;
  }();
  if (w.qmax <= 8 && ws && w.st == nullptr) return launch_ws<HD>(m, n_rows, g, q, w, out, s);
  if (w.qmax <= 8) return launch_t<HD, 1>(tm_k, tm_v, m, n_rows, g, q, w, out, s);
  if (mq_enabled()) {
    if (w.qmax <= 16) return launch_mq<HD, 2>(m, n_rows, g, q, w, out, s);
    return launch_mq<HD, 3>(m, n_rows, g, q, w, out, s);
  }
  if (w.qmax <= 16) return launch_t<HD, 2>(tm_k, tm_v, m, n_rows, g, q, w, out, s);
  return launch_t<HD, 3>(tm_k, tm_v, m, n_rows, g, q, w, out, s);
}

}  // namespace

int attn_ctas(int n_rows, int chunks, int heads, int qmax) {
  if (qmax <= kDecodeQ) return n_rows * std::max(1, chunks) * heads * 2;  // DecCfg::kCluster
  if (qmax > 8 && mq_enabled()) return n_rows * std::max(1, chunks) * heads;
  return (n_rows * std::max(1, chunks) * heads + kVW - 1) / kVW;
}

int attn_chunks(int rows, int heads, int num_sms, int qmax) {
  if (qmax <= kDecodeQ) {
    // attn_decode_kernel: one 4-warp CTA per item. Whole (request, head) pairs per CTA
    // unless there are too few of them to fill the SMs: a split-KV merge (gpu-scope
    // fence + arrival counter) costs more than the longer per-CTA chain.
    static const double cps = [] {
      const char* e = std::getenv("SPIN_ATTN_DEC_CPS");  // experiments only
      return e ? std::atof(e) : 1.0;
    }();
    const double want = cps * num_sms / std::max(1, rows * heads);
    return std::max(1, std::min(16, static_cast<int>(std::lround(want))));
  }
  // attn_kernel: ~8 warps of work per SM (2 CTAs x 4 warps): rows x chunks x heads ~= 8 x SMs
  static const double wps = [] {
    const char* e = std::getenv("SPIN_ATTN_WPS");  // experiments only
    return e ? std::atof(e) : 8.0;
  }();
  const double want = wps * num_sms / std::max(1, rows * heads);
  return std::max(1, std::min(16, static_cast<int>(std::lround(want))));
}

void launch_attention(const CUtensorMap& tm_k, const CUtensorMap& tm_v, const FwdMeta& m, int n_rows, int n_req,
                      const AttnGeom& g, const float* q, const AttnWork& w, bf16* out, cudaStream_t s) {
  (void)n_req;
  if (n_rows <= 0) return;
  if (w.qmax <= kDecodeQ) {
    if (g.head_dim == 128) return launch_decode<128>(m, n_rows, g, q, w, out, s);
    return launch_decode<64>(m, n_rows, g, q, w, out, s);
  }
  if (g.head_dim == 128) return launch_hd<128>(tm_k, tm_v, m, n_rows, g, q, w, out, s);
  return launch_hd<64>(tm_k, tm_v, m, n_rows, g, q, w, out, s);
}

}  // namespace spin
