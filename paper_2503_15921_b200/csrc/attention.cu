// Packed ragged causal attention for the verify / draft forward (K4 + K5).
//
// Work decomposition = the request decomposition of the reference packer
// (packing.cpp:16-103): CTA (pack row, head) walks the segments of its row;
// each segment is a contiguous key range of one request's KV cache. Instead of
// copying KV into a packed [W, L] tensor the kernel reads the per-slot cache in
// place (zero-copy packing); equal row lengths L give equal work per CTA.
//
// Per segment the request's queries (its verify rows) attend over the
// segment's keys with a causal mask on absolute positions; the segment emits
// (max, sum, unnormalised output) per query and the combine kernel merges the
// request's segments under one shared max -- the modified attention of
// attention.cpp:128-157 / PAPER.md:460-464, with scale 1/sqrt(hd) and causality.
//
// CTA = 4 consumer warps + 1 TMA producer warp. KV tiles of 32 keys are
// TMA-loaded (128-B swizzle, box 64 dims x 32 keys) into a ring of stages;
// consumer warp w takes tiles w, w+4, ... of each segment; lane = key for
// Q.K, lane = 4 (or 2) head dims for P.V, warp-shuffle online softmax.
#include "kernels.cuh"
#include "ptx.cuh"

namespace spin {

namespace {

constexpr int kConsumerWarps = 4;
constexpr int kAttnThreads = 32 * (kConsumerWarps + 1);
constexpr int kTileKeys = 32;
constexpr unsigned kFull = 0xffffffffu;

// Ring stages are owned per consumer warp (warp w consumes tiles w, w+4, ...
// from its own kPerWarp stages, in order): an mbarrier parity wait is then never
// more than one phase ahead of the stage it waits on.
template <int HD>
struct AttnCfg {
  static constexpr int kBoxes = HD / 64;                 // 64-dim (128-B) boxes per key row
  static constexpr int kTileBytes = kTileKeys * HD * 2;  // one of K or V
  static constexpr int kPerWarp = HD == 128 ? 1 : 2;     // 64 KB / 32 KB ring
  static constexpr int kStages = kConsumerWarps * kPerWarp;
  static constexpr int kDpl = HD / 32;                   // dims per lane in P.V
};

// tile t (CTA-global count) -> ring stage and phase
template <int HD>
__device__ __forceinline__ int tile_stage(int t) {
  return (t % kConsumerWarps) + kConsumerWarps * ((t / kConsumerWarps) % AttnCfg<HD>::kPerWarp);
}
template <int HD>
__device__ __forceinline__ uint32_t tile_phase(int t) {
  return static_cast<uint32_t>((t / AttnCfg<HD>::kStages) & 1);
}

template <int HD, int QMAX>
struct AttnSmem {
  static constexpr int kQPad = (QMAX + 3) / 4 * 4;  // p row stride (float4 reads)
  static constexpr size_t kRing = static_cast<size_t>(AttnCfg<HD>::kStages) * 2 * AttnCfg<HD>::kTileBytes;
  static constexpr size_t kQ = static_cast<size_t>(QMAX) * HD * 4;
  // per-warp p[key][query] buffers, reused as the segment merge buffer [QMAX][HD+2]
  static constexpr size_t kPBuf = static_cast<size_t>(kConsumerWarps) * kTileKeys * kQPad * 4;
  static constexpr size_t kMergeBuf = static_cast<size_t>(QMAX) * (HD + 2) * 4;
  static constexpr size_t kP = (kPBuf > kMergeBuf ? kPBuf : kMergeBuf + 15) / 16 * 16;
  static constexpr size_t kBars = 2 * 8 * 8;
  static constexpr size_t kTotal = 1024 + kRing + kQ + kP + kBars;
};

__device__ __forceinline__ uint64_t f2_bits(float2 v) { return *reinterpret_cast<uint64_t*>(&v); }
__device__ __forceinline__ float2 bits_f2(uint64_t v) { return *reinterpret_cast<float2*>(&v); }

// Blackwell packed fp32x2 FMA (FFMA2): two IEEE fp32 FMAs per instruction.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)), "l"(f2_bits(c)));
  return bits_f2(d);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return bits_f2(d);
}
// bf16 pair (packed in 32 bits) -> fp32 pair
__device__ __forceinline__ float2 bf2_to_f2(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}

template <int HD, int QMAX>
__global__ void __launch_bounds__(kAttnThreads) attention_kernel(const __grid_constant__ CUtensorMap tm_k,
                                                                 const __grid_constant__ CUtensorMap tm_v, FwdMeta m,
                                                                 AttnGeom g, const float* __restrict__ q, AttnWork w) {
  using Cfg = AttnCfg<HD>;
  using Sm = AttnSmem<HD, QMAX>;
  constexpr int S = Cfg::kStages;
  constexpr int DPL = Cfg::kDpl;
  constexpr int QP = Sm::kQPad;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint8_t* ring = smem;
  float* sq = reinterpret_cast<float*>(smem + Sm::kRing);
  float* sp_all = reinterpret_cast<float*>(smem + Sm::kRing + Sm::kQ);
  float* smerge = sp_all;  // aliases the p buffers: used only between segment barriers
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Sm::kRing + Sm::kQ + Sm::kP);
  uint64_t* empty_bar = full_bar + 8;

  const int prow = blockIdx.x, head = blockIdx.y;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int H = g.n_heads, D = H * HD;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  ptx::grid_dep_wait();

  const int seg_begin = m.row_ptr[prow], seg_end = m.row_ptr[prow + 1];

  if (warp == kConsumerWarps) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      const uint64_t pol = ptx::policy_evict_first();
      int gt = 0;
      for (int si = seg_begin; si < seg_end; ++si) {
        const int sid = m.row_seg[si];
        const int32_t* sg = m.seg + 5 * sid;
        const int rq = sg[0], len = sg[3] - sg[2], off = sg[4];
        const int slot = m.req_slot[rq];
        const int base = ((g.layer * g.slots + slot) * H + head) * g.ctx + off;
        const int ntiles = (len + kTileKeys - 1) / kTileKeys;
        for (int t = 0; t < ntiles; ++t, ++gt) {
          const int st = tile_stage<HD>(gt);
          ptx::mbar_wait(&empty_bar[st], tile_phase<HD>(gt) ^ 1);
          ptx::mbar_arrive_expect_tx(&full_bar[st], 2 * Cfg::kTileBytes);
          uint8_t* kdst = ring + static_cast<size_t>(st) * 2 * Cfg::kTileBytes;
          uint8_t* vdst = kdst + Cfg::kTileBytes;
#pragma unroll
          for (int b = 0; b < Cfg::kBoxes; ++b) {
#pragma unroll
            for (int hb = 0; hb < 2; ++hb) {  // tensor-map boxes are 16 keys x 64 dims (2 KiB)
              ptx::tma_load_2d(kdst + b * 4096 + hb * 2048, &tm_k, &full_bar[st], b * 64,
                               base + t * kTileKeys + hb * 16, pol);
              ptx::tma_load_2d(vdst + b * 4096 + hb * 2048, &tm_v, &full_bar[st], b * 64,
                               base + t * kTileKeys + hb * 16, pol);
            }
          }
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  float* sp = sp_all + warp * kTileKeys * QP;  // this warp's p[key][query]
  int gt = 0;
  for (int si = seg_begin; si < seg_end; ++si) {
    const int sid = m.row_seg[si];
    const int32_t* sg = m.seg + 5 * sid;
    const int rq = sg[0], len = sg[3] - sg[2], off = sg[4];
    const int qlen = m.req_qlen[rq], kvlen = m.req_kvlen[rq], qs = m.req_qstart[rq];
    const int ntiles = (len + kTileKeys - 1) / kTileKeys;

    // stage this request's queries for the head (fp32, zero beyond qlen)
    for (int e = threadIdx.x; e < QMAX * HD; e += 32 * kConsumerWarps) {
      const int j = e / HD, d = e % HD;
      sq[e] = j < qlen ? q[static_cast<size_t>(qs + j) * D + head * HD + d] : 0.f;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");

    float mrun[QMAX], lsum[QMAX];  // running max (warp-uniform), per-lane exp-sum
    float2 o[QMAX][DPL / 2];
#pragma unroll
    for (int j = 0; j < QMAX; ++j) {
      mrun[j] = -INFINITY;
      lsum[j] = 0.f;
#pragma unroll
      for (int d = 0; d < DPL / 2; ++d) o[j][d] = make_float2(0.f, 0.f);
    }

    // warp w owns the tiles whose CTA-global index gt+t is w mod 4 (its ring stages)
    for (int t = ((warp - gt) % kConsumerWarps + kConsumerWarps) % kConsumerWarps; t < ntiles;
         t += kConsumerWarps) {
      const int gi = gt + t;
      const int st = tile_stage<HD>(gi);
      ptx::mbar_wait(&full_bar[st], tile_phase<HD>(gi));
      const uint8_t* ks = ring + static_cast<size_t>(st) * 2 * Cfg::kTileBytes;
      const uint8_t* vs = ks + Cfg::kTileBytes;
      const int kidx = t * kTileKeys + lane;  // key index within the segment
      const int kpos = off + kidx;            // absolute position of this lane's key

      // ---- scores, lane = key: q.k in fp32 pairs (FFMA2)
      float2 acc[QMAX];
#pragma unroll
      for (int j = 0; j < QMAX; ++j) acc[j] = make_float2(0.f, 0.f);
#pragma unroll
      for (int c = 0; c < HD / 8; ++c) {
        const int box = c / 8, cc = c % 8;
        const uint4 kr = *reinterpret_cast<const uint4*>(ks + box * 4096 + lane * 128 + ((cc ^ (lane & 7)) << 4));
        const float2 k0 = bf2_to_f2(kr.x), k1 = bf2_to_f2(kr.y), k2 = bf2_to_f2(kr.z), k3 = bf2_to_f2(kr.w);
#pragma unroll
        for (int j = 0; j < QMAX; ++j) {
          if (j < qlen) {
            const float4 qa = *reinterpret_cast<const float4*>(sq + j * HD + c * 8);
            const float4 qb = *reinterpret_cast<const float4*>(sq + j * HD + c * 8 + 4);
            acc[j] = ffma2(make_float2(qa.x, qa.y), k0, acc[j]);
            acc[j] = ffma2(make_float2(qa.z, qa.w), k1, acc[j]);
            acc[j] = ffma2(make_float2(qb.x, qb.y), k2, acc[j]);
            acc[j] = ffma2(make_float2(qb.z, qb.w), k3, acc[j]);
          }
        }
      }
      // ---- online softmax: warp max per query, per-lane sums
#pragma unroll
      for (int j = 0; j < QMAX; ++j) {
        if (j < qlen) {
          const int qpos = kvlen - qlen + j;
          const float sc = (kidx < len && kpos <= qpos) ? (acc[j].x + acc[j].y) * g.scale : -INFINITY;
          float mx = sc;
#pragma unroll
          for (int ofs = 16; ofs > 0; ofs >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, ofs));
          const float mnew = fmaxf(mrun[j], mx);
          float corr = 1.f, pj = 0.f;
          if (mnew != -INFINITY) {
            corr = expf(mrun[j] - mnew);
            pj = expf(sc - mnew);
          }
          lsum[j] = lsum[j] * corr + pj;
          mrun[j] = mnew;
#pragma unroll
          for (int d = 0; d < DPL / 2; ++d) o[j][d] = fmul2(o[j][d], make_float2(corr, corr));
          sp[lane * QP + j] = pj;
        }
      }
      __syncwarp();
      // ---- P.V: lane owns DPL consecutive dims, p broadcast from shared memory
      const int dim0 = lane * DPL;
      const int box = dim0 / 64, col = dim0 % 64, chunk = col / 8, inb = (col % 8) * 2;
#pragma unroll 4
      for (int r = 0; r < kTileKeys; ++r) {
        const uint8_t* vp = vs + box * 4096 + r * 128 + ((chunk ^ (r & 7)) << 4) + inb;
        float2 v[DPL / 2];
        if constexpr (DPL == 4) {
          const uint2 u = *reinterpret_cast<const uint2*>(vp);
          v[0] = bf2_to_f2(u.x);
          v[1] = bf2_to_f2(u.y);
        } else {
          v[0] = bf2_to_f2(*reinterpret_cast<const uint32_t*>(vp));
        }
        float pr[QP];
#pragma unroll
        for (int j4 = 0; j4 < QP; j4 += 4) {
          const float4 p4 = *reinterpret_cast<const float4*>(sp + r * QP + j4);
          pr[j4] = p4.x, pr[j4 + 1] = p4.y, pr[j4 + 2] = p4.z, pr[j4 + 3] = p4.w;
        }
#pragma unroll
        for (int j = 0; j < QMAX; ++j) {
          if (j < qlen) {
#pragma unroll
            for (int d = 0; d < DPL / 2; ++d) o[j][d] = ffma2(make_float2(pr[j], pr[j]), v[d], o[j][d]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&empty_bar[st]);
    }
    gt += ntiles;

    // ---- merge the 4 warps' partial states in warp order (deterministic), then
    // emit the segment partial (max, sum, unnormalised output) per query.
    asm volatile("bar.sync 1, 128;" ::: "memory");  // p buffers become the merge buffer
    for (int ww = 0; ww < kConsumerWarps; ++ww) {
      if (warp == ww) {
#pragma unroll
        for (int j = 0; j < QMAX; ++j) {
          if (j < qlen) {
            float l = lsum[j];
#pragma unroll
            for (int ofs = 16; ofs > 0; ofs >>= 1) l += __shfl_xor_sync(kFull, l, ofs);
            float* b = smerge + j * (HD + 2);
            if (ww == 0) {
#pragma unroll
              for (int d = 0; d < DPL / 2; ++d) {
                b[lane * DPL + 2 * d] = o[j][d].x;
                b[lane * DPL + 2 * d + 1] = o[j][d].y;
              }
              if (lane == 0) b[HD] = mrun[j], b[HD + 1] = l;
            } else {
              const float mo = b[HD], M = fmaxf(mo, mrun[j]);
              const float fo = (M == -INFINITY || mo == -INFINITY) ? 0.f : expf(mo - M);
              const float fn = (M == -INFINITY || mrun[j] == -INFINITY) ? 0.f : expf(mrun[j] - M);
#pragma unroll
              for (int d = 0; d < DPL / 2; ++d) {
                float* bd = b + lane * DPL + 2 * d;
                bd[0] = bd[0] * fo + o[j][d].x * fn;
                bd[1] = bd[1] * fo + o[j][d].y * fn;
              }
              __syncwarp();
              if (lane == 0) b[HD] = M, b[HD + 1] = b[HD + 1] * fo + l * fn;
            }
          }
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    for (int e = threadIdx.x; e < qlen * HD; e += 32 * kConsumerWarps) {
      const int j = e / HD, d = e % HD;
      const float* b = smerge + j * (HD + 2);
      const size_t pi = (static_cast<size_t>(sid) * H + head) * w.qmax + j;
      w.part_o[pi * HD + d] = b[d];
      if (d == 0) {
        w.part_m[pi] = b[HD];
        w.part_l[pi] = b[HD + 1];
      }
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
  }
}

// ---------------------------------------------------------------------------
// Tensor-core variant (requests with <= 8 queries): mma.sync m16n8k16 bf16
// with fp32 accumulation, FlashAttention-2 register layout (the S accumulator
// fragment of two 8-key tiles is the P operand fragment of one 16-key step).
// Q is split 3-way (hi/mid/lo bf16, ~24 mantissa bits) and P 2-way, so scores
// and outputs keep ~fp32 accuracy. Each consumer warp owns its ring stage and
// writes its own (max, sum, output) partial per segment: no CTA barriers in the
// main loop; the combine kernel merges segments x warps under one shared max.
__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
  const uint32_t a = __bfloat16_as_ushort(__float2bfloat16_rn(lo));
  const uint32_t b = __bfloat16_as_ushort(__float2bfloat16_rn(hi));
  return a | (b << 16);
}
__device__ __forceinline__ float bf_round(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

__device__ __forceinline__ void mma_bf16(float& d0, float& d1, uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  float x2, x3;  // rows g+8 of the 16-row tile: padding queries, discarded
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%10,%11,%12,%13};"
      : "=f"(d0), "=f"(d1), "=f"(x2), "=f"(x3)
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1), "f"(d0), "f"(d1), "f"(0.f), "f"(0.f));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

// byte offset of (key row, 16-B chunk) inside a TMA 128-B-swizzled KV tile
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return static_cast<uint32_t>((chunk >> 3) * 4096 + row * 128 + (((chunk & 7) ^ (row & 7)) << 4));
}

constexpr int kMmaSub = kConsumerWarps;  // partials per (segment, head)

constexpr int kMmaKeys = 16;  // keys per tile in the tensor-core kernel (one 16-row TMA box)

template <int HD>
struct MmaSmem {
  static constexpr uint32_t kHalf = kMmaKeys * HD * 2;         // K or V of one tile (4 KiB at HD 128)
  static constexpr uint32_t kStage = 2 * kHalf;                // K + V
  static constexpr uint32_t kWarpRing = 2 * kStage;            // double buffer per consumer warp
  static constexpr size_t kRing = static_cast<size_t>(kConsumerWarps) * kWarpRing;
  static constexpr uint32_t kQPlane = 8 * HD * 2;              // 8 query rows, bf16
  static constexpr uint32_t kSlot = 3 * kQPlane + 64;          // hi/mid/lo planes + segment header
  static constexpr uint32_t kMerge = kConsumerWarps * 8 * (HD + 2) * 4;  // per-warp partials of a segment
  static constexpr size_t kTotal = 1024 + kRing + 2 * kSlot + 2 * kMerge + 16 * 8 + 16;
};

// byte offset of (row, 16-B chunk) in a Q plane with HD*2-byte rows, chunks XOR-swizzled by row
template <int HD>
__device__ __forceinline__ uint32_t qswz(int row, int chunk) {
  return static_cast<uint32_t>(row * HD * 2 + (((chunk & 7) ^ (row & 7)) | (chunk & ~7)) * 16);
}
// byte offset of (key row, 16-B chunk) in a 16-key TMA tile: 64-dim boxes of 2 KiB
__device__ __forceinline__ uint32_t kswz(int row, int chunk) {
  return static_cast<uint32_t>((chunk >> 3) * 2048 + row * 128 + (((chunk & 7) ^ (row & 7)) << 4));
}

// Segment header staged by the producer warp
struct SegHdr {
  int sid, len, off, qlen, kvlen, qs, slot, pad;
};

template <int HD>
__global__ void __launch_bounds__(kAttnThreads) attention_mma_kernel(const __grid_constant__ CUtensorMap tm_k,
                                                                     const __grid_constant__ CUtensorMap tm_v,
                                                                     FwdMeta m, AttnGeom g,
                                                                     const float* __restrict__ q, AttnWork w) {
  using Sm = MmaSmem<HD>;
  constexpr int KS = HD / 16;  // 16-dim k-steps
  constexpr int DN = HD / 8;   // 8-dim output tiles
  constexpr int kBoxes = HD / 64;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint8_t* slots = smem + Sm::kRing;  // 2 x {3 Q planes, header}
  float* merge = reinterpret_cast<float*>(slots + 2 * Sm::kSlot);  // 2 x [warp][8][HD+2]
  uint64_t* bars = reinterpret_cast<uint64_t*>(slots + 2 * Sm::kSlot + 2 * Sm::kMerge);
  uint64_t* qfull_bar = bars;        // [2]
  uint64_t* qempty_bar = bars + 2;   // [2]
  uint64_t* kv_bar = bars + 4;       // [warp][2]
  int* merge_count = reinterpret_cast<int*>(bars + 4 + 2 * kConsumerWarps);  // [2]

  const int prow = blockIdx.x, head = blockIdx.y;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int g8 = lane >> 2, c4 = lane & 3;
  const int H = g.n_heads, D = H * HD;

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&qfull_bar[s], 1);
      ptx::mbar_init(&qempty_bar[s], kConsumerWarps);
    }
    for (int s = 0; s < 2 * kConsumerWarps; ++s) ptx::mbar_init(&kv_bar[s], 1);
    merge_count[0] = merge_count[1] = 0;
    ptx::fence_mbar_init();
  }
  __syncthreads();
  ptx::grid_dep_wait();
  const int seg_begin = m.row_ptr[prow], nseg = m.row_ptr[prow + 1] - seg_begin;

  if (warp == kConsumerWarps) {
    // ------------------------------------------------------------ producer warp:
    // stages each segment's header and split Q planes, up to 2 segments ahead.
    for (int k = 0; k < nseg; ++k) {
      const int sid = m.row_seg[seg_begin + k];
      const int32_t* sg = m.seg + 5 * sid;
      const int rq = sg[0];
      const int qlen = m.req_qlen[rq], qs = m.req_qstart[rq];
      const int sl = k & 1;
      uint8_t* slot = slots + sl * Sm::kSlot;
      ptx::mbar_wait(&qempty_bar[sl], ((k >> 1) & 1) ^ 1);
      const uint32_t qp = ptx::smem_u32(slot);
      for (int e = lane; e < 8 * HD / 8; e += 32) {  // one 16-B chunk (8 dims) per step
        const int row = e / (HD / 8), chunk = e % (HD / 8);
        float x[8];
        if (row < qlen) {
          const float4* src =
              reinterpret_cast<const float4*>(q + static_cast<size_t>(qs + row) * D + head * HD + chunk * 8);
          const float4 a = src[0], b = src[1];
          x[0] = a.x, x[1] = a.y, x[2] = a.z, x[3] = a.w, x[4] = b.x, x[5] = b.y, x[6] = b.z, x[7] = b.w;
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) x[i] = 0.f;
        }
        uint32_t hi[4], mi[4], lo[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float h0 = bf_round(x[2 * i]), h1 = bf_round(x[2 * i + 1]);
          const float r0 = x[2 * i] - h0, r1 = x[2 * i + 1] - h1;
          const float m0 = bf_round(r0), m1 = bf_round(r1);
          hi[i] = pack_bf2(h0, h1);
          mi[i] = pack_bf2(m0, m1);
          lo[i] = pack_bf2(r0 - m0, r1 - m1);
        }
        const uint32_t o = qswz<HD>(row, chunk);
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(qp + o), "r"(hi[0]), "r"(hi[1]), "r"(hi[2]),
                     "r"(hi[3]));
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(qp + Sm::kQPlane + o), "r"(mi[0]), "r"(mi[1]),
                     "r"(mi[2]), "r"(mi[3]));
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(qp + 2 * Sm::kQPlane + o), "r"(lo[0]),
                     "r"(lo[1]), "r"(lo[2]), "r"(lo[3]));
      }
      if (lane == 0) {
        SegHdr* hdr = reinterpret_cast<SegHdr*>(slot + 3 * Sm::kQPlane);
        hdr->sid = sid, hdr->len = sg[3] - sg[2], hdr->off = sg[4], hdr->qlen = qlen;
        hdr->kvlen = m.req_kvlen[rq], hdr->qs = qs, hdr->slot = m.req_slot[rq];
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&qfull_bar[sl]);  // release: planes + header visible
    }
    return;
  }

  // -------------------------------------------------------------- consumer warps
  // Each warp computes tiles t = warp, warp+4, ... of every segment, double
  // buffering its own 16-key K/V tiles (lane 0 issues the TMA), looking at most
  // one segment ahead so that it never needs a Q slot it still holds.
  if (nseg == 0) return;
  uint8_t* ring = smem + static_cast<size_t>(warp) * Sm::kWarpRing;
  uint64_t* bar = kv_bar + 2 * warp;
  const uint64_t pol = ptx::policy_evict_first();
  auto header = [&](int k) {
    ptx::mbar_wait(&qfull_bar[k & 1], (k >> 1) & 1);
    return *reinterpret_cast<const SegHdr*>(slots + (k & 1) * Sm::kSlot + 3 * Sm::kQPlane);
  };
  auto tiles_of = [](const SegHdr& h) { return (h.len + kMmaKeys - 1) / kMmaKeys; };

  int ck = 0;
  SegHdr cur = header(0), nxt{};
  bool have_nxt = false;
  // issue iterator
  int ik = 0, it = warp, issued = 0, consumed = 0;
  auto try_issue = [&]() {
    while (issued - consumed < 2) {
      const SegHdr* ih = ik == ck ? &cur : &nxt;
      while (it >= tiles_of(*ih)) {  // advance to the next segment with a tile for this warp
        if (ik + 1 >= nseg || ik + 1 > ck + 1) return;
        ++ik;
        it = warp;
        if (!have_nxt) {
          nxt = header(ik);
          have_nxt = true;
        }
        ih = &nxt;
      }
      if (lane == 0) {
        const int st = issued & 1;
        uint8_t* dst = ring + st * Sm::kStage;
        const int row0 = ((g.layer * g.slots + ih->slot) * H + head) * g.ctx + ih->off + it * kMmaKeys;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        ptx::mbar_arrive_expect_tx(&bar[st], Sm::kStage);
#pragma unroll
        for (int b = 0; b < kBoxes; ++b) {
          ptx::tma_load_2d(dst + b * 2048, &tm_k, &bar[st], b * 64, row0, pol);
          ptx::tma_load_2d(dst + Sm::kHalf + b * 2048, &tm_v, &bar[st], b * 64, row0, pol);
        }
      }
      ++issued;
      it += kConsumerWarps;
    }
  };
  try_issue();

  while (true) {
    const int len = cur.len, off = cur.off, qlen = cur.qlen;
    const bool qrow = g8 < qlen;
    const int qpos = cur.kvlen - qlen + g8;
    const uint32_t qp_base = ptx::smem_u32(slots + (ck & 1) * Sm::kSlot);
    float mrun = -INFINITY, lsum = 0.f;
    float2 o[DN];
#pragma unroll
    for (int dn = 0; dn < DN; ++dn) o[dn] = make_float2(0.f, 0.f);

    for (int t = warp; t < tiles_of(cur); t += kConsumerWarps) {
      const int st = consumed & 1;
      ptx::mbar_wait(&bar[st], (consumed >> 1) & 1);
      const uint32_t ks_base = ptx::smem_u32(ring + st * Sm::kStage);
      const uint32_t vs_base = ks_base + Sm::kHalf;
      // ---- S = Q K^T for 2 tiles of 8 keys, 32 dims (two k-steps) at a time
      float s[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
      for (int kp = 0; kp < KS / 2; ++kp) {
        uint32_t qa[3][4];
        const uint32_t qoff = qswz<HD>(lane & 7, kp * 4 + (lane >> 3));
#pragma unroll
        for (int sp = 0; sp < 3; ++sp)
          ldsm_x4(qp_base + sp * Sm::kQPlane + qoff, qa[sp][0], qa[sp][1], qa[sp][2], qa[sp][3]);
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4(ks_base + kswz(n * 8 + (lane & 7), kp * 4 + (lane >> 3)), b0, b1, b2, b3);
#pragma unroll
          for (int sp = 0; sp < 3; ++sp) {
            mma_bf16(s[n][0], s[n][1], qa[sp][0], qa[sp][1], b0, b1);
            mma_bf16(s[n][0], s[n][1], qa[sp][2], qa[sp][3], b2, b3);
          }
        }
      }
      // ---- online softmax on row g8 (quad reduction)
      float tmax = -INFINITY;
#pragma unroll
      for (int n = 0; n < 2; ++n) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int kidx = t * kMmaKeys + n * 8 + 2 * c4 + e;
          const bool ok = qrow && kidx < len && off + kidx <= qpos;
          s[n][e] = ok ? s[n][e] * g.scale : -INFINITY;
          tmax = fmaxf(tmax, s[n][e]);
        }
      }
      tmax = fmaxf(tmax, __shfl_xor_sync(kFull, tmax, 1));
      tmax = fmaxf(tmax, __shfl_xor_sync(kFull, tmax, 2));
      const float mnew = fmaxf(mrun, tmax);
      const float corr = mnew == -INFINITY ? 1.f : expf(mrun - mnew);
#pragma unroll
      for (int n = 0; n < 2; ++n) {
#pragma unroll
        for (int e = 0; e < 2; ++e) s[n][e] = mnew == -INFINITY ? 0.f : expf(s[n][e] - mnew);
      }
      lsum = lsum * corr + (s[0][0] + s[0][1]) + (s[1][0] + s[1][1]);
      mrun = mnew;
#pragma unroll
      for (int dn = 0; dn < DN; ++dn) o[dn] = fmul2(o[dn], make_float2(corr, corr));
      // ---- O += P V (16 keys), P split 2-way
      {
        const float h00 = bf_round(s[0][0]), h01 = bf_round(s[0][1]), h10 = bf_round(s[1][0]),
                    h11 = bf_round(s[1][1]);
        const uint32_t ah0 = pack_bf2(h00, h01), ah2 = pack_bf2(h10, h11);
        const uint32_t al0 = pack_bf2(s[0][0] - h00, s[0][1] - h01), al2 = pack_bf2(s[1][0] - h10, s[1][1] - h11);
        const int vrow = ((lane >> 3) & 1) * 8 + (lane & 7);
#pragma unroll
        for (int dp = 0; dp < DN / 2; ++dp) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(vs_base + kswz(vrow, dp * 2 + (lane >> 4)), b0, b1, b2, b3);
          mma_bf16(o[2 * dp].x, o[2 * dp].y, ah0, ah2, b0, b1);
          mma_bf16(o[2 * dp].x, o[2 * dp].y, al0, al2, b0, b1);
          mma_bf16(o[2 * dp + 1].x, o[2 * dp + 1].y, ah0, ah2, b2, b3);
          mma_bf16(o[2 * dp + 1].x, o[2 * dp + 1].y, al0, al2, b2, b3);
        }
      }
      ++consumed;
      __syncwarp();
      try_issue();
    }
    // ---- this warp's partial for the segment; the last warp to finish merges
    // the 4 partials in warp order (deterministic) and writes one per segment.
    lsum += __shfl_xor_sync(kFull, lsum, 1);
    lsum += __shfl_xor_sync(kFull, lsum, 2);
    float* mb = merge + (ck & 1) * (Sm::kMerge / 4);
    {
      float* mine = mb + (warp * 8 + g8) * (HD + 2);
#pragma unroll
      for (int dn = 0; dn < DN; ++dn) *reinterpret_cast<float2*>(mine + dn * 8 + 2 * c4) = o[dn];
      if (c4 == 0) mine[HD] = mrun, mine[HD + 1] = lsum;
    }
    __threadfence_block();
    __syncwarp();
    int last = 0;
    if (lane == 0) last = atomicAdd(&merge_count[ck & 1], 1) == kConsumerWarps - 1;
    last = __shfl_sync(kFull, last, 0);
    if (last) {
      __threadfence_block();
      if (qrow) {
        float M = -INFINITY;
#pragma unroll
        for (int ww = 0; ww < kConsumerWarps; ++ww) M = fmaxf(M, mb[(ww * 8 + g8) * (HD + 2) + HD]);
        float f[kConsumerWarps], L = 0.f;
#pragma unroll
        for (int ww = 0; ww < kConsumerWarps; ++ww) {
          const float mw = mb[(ww * 8 + g8) * (HD + 2) + HD];
          f[ww] = mw == -INFINITY ? 0.f : expf(mw - M);
          L += mb[(ww * 8 + g8) * (HD + 2) + HD + 1] * f[ww];
        }
        const size_t pi = (static_cast<size_t>(cur.sid) * H + head) * w.qmax + g8;
#pragma unroll
        for (int dn = 0; dn < DN; ++dn) {
          float2 acc = make_float2(0.f, 0.f);
#pragma unroll
          for (int ww = 0; ww < kConsumerWarps; ++ww) {
            if (f[ww] == 0.f) continue;
            const float2 v = *reinterpret_cast<const float2*>(mb + (ww * 8 + g8) * (HD + 2) + dn * 8 + 2 * c4);
            acc.x += v.x * f[ww];
            acc.y += v.y * f[ww];
          }
          *reinterpret_cast<float2*>(w.part_o + pi * HD + dn * 8 + 2 * c4) = acc;
        }
        if (c4 == 0) w.part_m[pi] = M, w.part_l[pi] = L;
      }
      __syncwarp();
      if (lane == 0) merge_count[ck & 1] = 0;
    }
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&qempty_bar[ck & 1]);  // done with this slot (Q planes, merge area)
    if (++ck >= nseg) break;
    cur = have_nxt ? nxt : header(ck);
    have_nxt = false;
    try_issue();
  }
}

// Shared-max merge of a request's segment partials (attention.cpp:134-157):
// M = max over partials, out = sum_p exp(m_p - M) o_p / sum_p exp(m_p - M) l_p.
// The (partial, query) weights are staged in shared memory in parallel, then
// every thread (one output dim) sums its column; fixed order = deterministic.
constexpr int kCombineMax = 512;  // partials x queries staged per block

template <int HD>
__global__ void attn_combine_kernel(FwdMeta m, AttnWork w, int H, int sub, bf16* out) {
  __shared__ float s_f[kCombineMax];
  __shared__ float s_inv[32];
  ptx::grid_dep_wait();
  const int rq = blockIdx.x, head = blockIdx.y, d = threadIdx.x;
  const int s0 = m.req_seg0[rq], ns = m.req_nseg[rq], qlen = m.req_qlen[rq], qs = m.req_qstart[rq];
  const int np = ns * sub;  // partials, ordered (segment, sub-partial)
  auto pidx = [&](int p, int j) {
    return ((static_cast<size_t>(s0 + p / sub) * H + head) * sub + p % sub) * w.qmax + j;
  };
  if (np * qlen <= kCombineMax && qlen <= 32) {
    // weights f[p][j] = exp(m_pj - M_j); one warp per query for the max / sum
    for (int e = threadIdx.x; e < np * qlen; e += blockDim.x) s_f[e] = w.part_m[pidx(e / qlen, e % qlen)];
    __syncthreads();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
    for (int j = warp; j < qlen; j += nw) {
      float M = -INFINITY;
      for (int p = lane; p < np; p += 32) M = fmaxf(M, s_f[p * qlen + j]);
      for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
      float L = 0.f;
      for (int p = lane; p < np; p += 32) {
        const float mp = s_f[p * qlen + j];
        const float f = mp == -INFINITY ? 0.f : expf(mp - M);
        L += w.part_l[pidx(p, j)] * f;
        s_f[p * qlen + j] = f;
      }
      for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
      if (lane == 0) s_inv[j] = 1.0f / L;
    }
    __syncthreads();
    for (int j = 0; j < qlen; ++j) {
      float O = 0.f;
#pragma unroll 4
      for (int p = 0; p < np; ++p) {
        const float f = s_f[p * qlen + j];
        const float v = f != 0.f ? __ldg(w.part_o + pidx(p, j) * HD + d) : 0.f;
        O += v * f;
      }
      out[static_cast<size_t>(qs + j) * H * HD + head * HD + d] = __float2bfloat16_rn(O * s_inv[j]);
    }
  } else {  // many partials (very long splits): direct two-pass form
    for (int j = 0; j < qlen; ++j) {
      float M = -INFINITY;
      for (int p = 0; p < np; ++p) M = fmaxf(M, w.part_m[pidx(p, j)]);
      float L = 0.f, O = 0.f;
      for (int p = 0; p < np; ++p) {
        const float mp = w.part_m[pidx(p, j)];
        if (mp == -INFINITY) continue;
        const float f = expf(mp - M);
        L += w.part_l[pidx(p, j)] * f;
        O += w.part_o[pidx(p, j) * HD + d] * f;
      }
      out[static_cast<size_t>(qs + j) * H * HD + head * HD + d] = __float2bfloat16_rn(O / L);
    }
  }
  ptx::grid_dep_launch();
}

template <int HD, int QMAX>
void launch_attn_t(const CUtensorMap& tm_k, const CUtensorMap& tm_v, const FwdMeta& m, int n_rows, int n_req,
                   const AttnGeom& g, const float* q, const AttnWork& w, bf16* out, cudaStream_t s) {
  using Sm = AttnSmem<HD, QMAX>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(attention_kernel<HD, QMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(Sm::kTotal));
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.stream = s;
  cfg.gridDim = dim3(n_rows, g.n_heads);
  cfg.blockDim = dim3(kAttnThreads);
  cfg.dynamicSmemBytes = Sm::kTotal;
  AttnWork ww = w;
  ww.qmax = QMAX;
  cudaLaunchKernelEx(&cfg, attention_kernel<HD, QMAX>, tm_k, tm_v, m, g, q, ww);
  cfg.gridDim = dim3(n_req, g.n_heads);
  cfg.blockDim = dim3(HD);
  cfg.dynamicSmemBytes = 0;
  cudaLaunchKernelEx(&cfg, attn_combine_kernel<HD>, m, ww, g.n_heads, 1, out);
}

template <int HD>
void launch_attn_mma(const CUtensorMap& tm_k, const CUtensorMap& tm_v, const FwdMeta& m, int n_rows, int n_req,
                     const AttnGeom& g, const float* q, const AttnWork& w, bf16* out, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(attention_mma_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(MmaSmem<HD>::kTotal));
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.stream = s;
  cfg.gridDim = dim3(n_rows, g.n_heads);
  cfg.blockDim = dim3(kAttnThreads);
  cfg.dynamicSmemBytes = MmaSmem<HD>::kTotal;
  AttnWork ww = w;
  ww.qmax = 8;
  cudaLaunchKernelEx(&cfg, attention_mma_kernel<HD>, tm_k, tm_v, m, g, q, ww);
  cfg.gridDim = dim3(n_req, g.n_heads);
  cfg.blockDim = dim3(HD);
  cfg.dynamicSmemBytes = 0;
  cudaLaunchKernelEx(&cfg, attn_combine_kernel<HD>, m, ww, g.n_heads, 1, out);
}

}  // namespace

void launch_attention(const CUtensorMap& tm_k, const CUtensorMap& tm_v, const FwdMeta& m, int n_rows, int n_req,
                      const AttnGeom& g, const float* q, const AttnWork& w, bf16* out, cudaStream_t s) {
  // w.qmax = the largest query count per request: <= 8 runs on the tensor
  // cores (mma.sync), 9..17 on the CUDA-core kernel.
  if (g.head_dim == 128) {
    if (w.qmax <= 8) return launch_attn_mma<128>(tm_k, tm_v, m, n_rows, n_req, g, q, w, out, s);
    return launch_attn_t<128, 17>(tm_k, tm_v, m, n_rows, n_req, g, q, w, out, s);
  }
  if (w.qmax <= 8) return launch_attn_mma<64>(tm_k, tm_v, m, n_rows, n_req, g, q, w, out, s);
  return launch_attn_t<64, 17>(tm_k, tm_v, m, n_rows, n_req, g, q, w, out, s);
}

int attention_qmax_bucket(int qmax) { return qmax <= 2 ? 2 : (qmax <= 8 ? 8 : 17); }

}  // namespace spin
