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

template <int HD>
struct AttnCfg {
  static constexpr int kBoxes = HD / 64;                 // 64-dim (128-B) boxes per key row
  static constexpr int kTileBytes = kTileKeys * HD * 2;  // one of K or V
  static constexpr int kStages = HD == 128 ? 4 : 6;
  static constexpr int kDpl = HD / 32;  // dims per lane in P.V
};

template <int HD, int QMAX>
struct AttnSmem {
  static constexpr size_t kRing = static_cast<size_t>(AttnCfg<HD>::kStages) * 2 * AttnCfg<HD>::kTileBytes;
  static constexpr size_t kQ = static_cast<size_t>(QMAX) * HD * 4;
  static constexpr size_t kMerge = static_cast<size_t>(kConsumerWarps) * QMAX * (HD + 2) * 4;
  static constexpr size_t kBars = 2 * 8 * 8;
  static constexpr size_t kTotal = 1024 + kRing + kQ + kMerge + kBars;
};

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

template <int HD, int QMAX>
__global__ void __launch_bounds__(kAttnThreads) attention_kernel(const __grid_constant__ CUtensorMap tm_k,
                                                                 const __grid_constant__ CUtensorMap tm_v, FwdMeta m,
                                                                 AttnGeom g, const float* __restrict__ q, AttnWork w) {
  using Cfg = AttnCfg<HD>;
  using Sm = AttnSmem<HD, QMAX>;
  constexpr int S = Cfg::kStages;
  constexpr int DPL = Cfg::kDpl;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint8_t* ring = smem;
  float* sq = reinterpret_cast<float*>(smem + Sm::kRing);
  float* smerge = reinterpret_cast<float*>(smem + Sm::kRing + Sm::kQ);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Sm::kRing + Sm::kQ + Sm::kMerge);
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
          const int st = gt % S;
          ptx::mbar_wait(&empty_bar[st], ((gt / S) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&full_bar[st], 2 * Cfg::kTileBytes);
          uint8_t* kdst = ring + static_cast<size_t>(st) * 2 * Cfg::kTileBytes;
          uint8_t* vdst = kdst + Cfg::kTileBytes;
#pragma unroll
          for (int b = 0; b < Cfg::kBoxes; ++b) {
            ptx::tma_load_2d(kdst + b * 4096, &tm_k, &full_bar[st], b * 64, base + t * kTileKeys, pol);
            ptx::tma_load_2d(vdst + b * 4096, &tm_v, &full_bar[st], b * 64, base + t * kTileKeys, pol);
          }
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
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

    float mrun[QMAX], lrun[QMAX], o[QMAX][DPL];
#pragma unroll
    for (int j = 0; j < QMAX; ++j) {
      mrun[j] = -INFINITY;
      lrun[j] = 0.f;
#pragma unroll
      for (int d = 0; d < DPL; ++d) o[j][d] = 0.f;
    }

    for (int t = warp; t < ntiles; t += kConsumerWarps) {
      const int gi = gt + t;
      const int st = gi % S;
      ptx::mbar_wait(&full_bar[st], (gi / S) & 1);
      const uint8_t* ks = ring + static_cast<size_t>(st) * 2 * Cfg::kTileBytes;
      const uint8_t* vs = ks + Cfg::kTileBytes;
      const int kidx = t * kTileKeys + lane;  // key index within the segment
      const int kpos = off + kidx;            // absolute position of this lane's key

      // ---- scores: lane = key
      float s[QMAX];
#pragma unroll
      for (int j = 0; j < QMAX; ++j) s[j] = 0.f;
#pragma unroll
      for (int c = 0; c < HD / 8; ++c) {
        const int box = c / 8, cc = c % 8;
        const uint4 raw8 = *reinterpret_cast<const uint4*>(ks + box * 4096 + lane * 128 + ((cc ^ (lane & 7)) << 4));
        float kf[8];
        bf16x8_to_f32(raw8, kf);
#pragma unroll
        for (int j = 0; j < QMAX; ++j) {
          if (j < qlen) {
            const float4 qa = *reinterpret_cast<const float4*>(sq + j * HD + c * 8);
            const float4 qb = *reinterpret_cast<const float4*>(sq + j * HD + c * 8 + 4);
            s[j] += qa.x * kf[0] + qa.y * kf[1] + qa.z * kf[2] + qa.w * kf[3] + qb.x * kf[4] + qb.y * kf[5] +
                    qb.z * kf[6] + qb.w * kf[7];
          }
        }
      }
      // ---- online softmax per query (warp-shuffle max / sum)
      float p[QMAX];
#pragma unroll
      for (int j = 0; j < QMAX; ++j) {
        p[j] = 0.f;
        if (j < qlen) {
          const int qpos = kvlen - qlen + j;
          const float sc = (kidx < len && kpos <= qpos) ? s[j] * g.scale : -INFINITY;
          float mx = sc;
#pragma unroll
          for (int ofs = 16; ofs > 0; ofs >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, ofs));
          const float mnew = fmaxf(mrun[j], mx);
          float corr = 1.f, pj = 0.f;
          if (mnew != -INFINITY) {
            corr = expf(mrun[j] - mnew);
            pj = expf(sc - mnew);
          }
          float ps = pj;
#pragma unroll
          for (int ofs = 16; ofs > 0; ofs >>= 1) ps += __shfl_xor_sync(kFull, ps, ofs);
          lrun[j] = lrun[j] * corr + ps;
          mrun[j] = mnew;
#pragma unroll
          for (int d = 0; d < DPL; ++d) o[j][d] *= corr;
          p[j] = pj;
        }
      }
      // ---- P.V: lane owns DPL consecutive dims
      const int dim0 = lane * DPL;
      const int box = dim0 / 64, col = dim0 % 64, chunk = col / 8, inb = (col % 8) * 2;
#pragma unroll 4
      for (int r = 0; r < kTileKeys; ++r) {
        const uint8_t* vp = vs + box * 4096 + r * 128 + ((chunk ^ (r & 7)) << 4) + inb;
        float vf[DPL];
        if constexpr (DPL == 4) {
          const uint2 u = *reinterpret_cast<const uint2*>(vp);
          vf[0] = __uint_as_float(u.x << 16);
          vf[1] = __uint_as_float(u.x & 0xffff0000u);
          vf[2] = __uint_as_float(u.y << 16);
          vf[3] = __uint_as_float(u.y & 0xffff0000u);
        } else {
          const uint32_t u = *reinterpret_cast<const uint32_t*>(vp);
          vf[0] = __uint_as_float(u << 16);
          vf[1] = __uint_as_float(u & 0xffff0000u);
        }
#pragma unroll
        for (int j = 0; j < QMAX; ++j) {
          if (j < qlen) {
            const float pr = __shfl_sync(kFull, p[j], r);
#pragma unroll
            for (int d = 0; d < DPL; ++d) o[j][d] += pr * vf[d];
          }
        }
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&empty_bar[st]);
    }
    gt += ntiles;

    // ---- merge the 4 warps' partial states, emit the segment partial
    float* mw = smerge + static_cast<size_t>(warp) * QMAX * (HD + 2);
#pragma unroll
    for (int j = 0; j < QMAX; ++j) {
      if (j < qlen) {
#pragma unroll
        for (int d = 0; d < DPL; ++d) mw[j * (HD + 2) + lane * DPL + d] = o[j][d];
        if (lane == 0) {
          mw[j * (HD + 2) + HD] = mrun[j];
          mw[j * (HD + 2) + HD + 1] = lrun[j];
        }
      }
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    for (int e = threadIdx.x; e < qlen * HD; e += 32 * kConsumerWarps) {
      const int j = e / HD, d = e % HD;
      float M = -INFINITY;
#pragma unroll
      for (int ww = 0; ww < kConsumerWarps; ++ww) M = fmaxf(M, smerge[(ww * QMAX + j) * (HD + 2) + HD]);
      float O = 0.f, L = 0.f;
#pragma unroll
      for (int ww = 0; ww < kConsumerWarps; ++ww) {
        const float* b = smerge + (ww * QMAX + j) * (HD + 2);
        const float f = (M == -INFINITY || b[HD] == -INFINITY) ? 0.f : expf(b[HD] - M);
        O += b[d] * f;
        L += b[HD + 1] * f;
      }
      const size_t pi = (static_cast<size_t>(sid) * H + head) * w.qmax + j;
      w.part_o[pi * HD + d] = O;
      if (d == 0) {
        w.part_m[pi] = M;
        w.part_l[pi] = L;
      }
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
  }
}

// Shared-max merge of a request's segment partials (attention.cpp:134-157).
template <int HD>
__global__ void attn_combine_kernel(FwdMeta m, AttnWork w, int H, bf16* out) {
  ptx::grid_dep_wait();
  const int rq = blockIdx.x, head = blockIdx.y, d = threadIdx.x;
  const int s0 = m.req_seg0[rq], ns = m.req_nseg[rq], qlen = m.req_qlen[rq], qs = m.req_qstart[rq];
  for (int j = 0; j < qlen; ++j) {
    float M = -INFINITY;
    for (int s = s0; s < s0 + ns; ++s) M = fmaxf(M, w.part_m[(static_cast<size_t>(s) * H + head) * w.qmax + j]);
    float L = 0.f, O = 0.f;
    for (int s = s0; s < s0 + ns; ++s) {
      const size_t pi = (static_cast<size_t>(s) * H + head) * w.qmax + j;
      const float ms = w.part_m[pi];
      const float f = ms == -INFINITY ? 0.f : expf(ms - M);
      L += w.part_l[pi] * f;
      O += w.part_o[pi * HD + d] * f;
    }
    out[static_cast<size_t>(qs + j) * H * HD + head * HD + d] = __float2bfloat16_rn(O / L);
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
  cudaLaunchKernelEx(&cfg, attn_combine_kernel<HD>, m, ww, g.n_heads, out);
}

}  // namespace

void launch_attention(const CUtensorMap& tm_k, const CUtensorMap& tm_v, const FwdMeta& m, int n_rows, int n_req,
                      const AttnGeom& g, const float* q, const AttnWork& w, bf16* out, cudaStream_t s) {
  // w.qmax selects the instantiation: the largest query count per request.
  if (g.head_dim == 128) {
    if (w.qmax <= 2) return launch_attn_t<128, 2>(tm_k, tm_v, m, n_rows, n_req, g, q, w, out, s);
    if (w.qmax <= 8) return launch_attn_t<128, 8>(tm_k, tm_v, m, n_rows, n_req, g, q, w, out, s);
    return launch_attn_t<128, 17>(tm_k, tm_v, m, n_rows, n_req, g, q, w, out, s);
  }
  if (w.qmax <= 2) return launch_attn_t<64, 2>(tm_k, tm_v, m, n_rows, n_req, g, q, w, out, s);
  if (w.qmax <= 8) return launch_attn_t<64, 8>(tm_k, tm_v, m, n_rows, n_req, g, q, w, out, s);
  return launch_attn_t<64, 17>(tm_k, tm_v, m, n_rows, n_req, g, q, w, out, s);
}

int attention_qmax_bucket(int qmax) { return qmax <= 2 ? 2 : (qmax <= 8 ? 8 : 17); }

}  // namespace spin
