// Fused projections of the SSM draft step (few token rows, T <= 32).
//
// A draft step of a 68M/160M SSM runs 12 x 8 kernels over 16..32 token rows;
// every kernel is latency-bound (a 160M layer is 19 MB of weights, ~3 us of
// HBM time over all SMs), so the step costs launches and dependent L2 round
// trips, not bytes. These kernels cut a layer from eight launches to five and
// each launch to about one round trip:
//
//   * one CTA per unit of 16 (or 32) output rows over the FULL K, so no split-K
//     partials and no separate reduction kernel: the epilogue (RoPE + KV append,
//     SwiGLU, residual add) runs in the projection itself;
//   * the unit's weight slab (rows x K, bf16, read from the tiled layout of
//     gemm.cuh as 1-KB row groups) is bulk-copied into shared memory BEFORE the
//     programmatic-dependent-launch wait, overlapping the previous kernel;
//   * RMSNorm is folded into the consumers: residual producers also write each
//     unit's sum of squares per token (ssp[t][unit], a token's partials contiguous);
//     a consumer multiplies with bf16(h) and scales each token's outputs by
//     1/rms(h) (a per-token factor of the product) computed from those sums in a
//     fixed order, so no normalised copy of the activations is materialised and
//     the matmul never waits on the sums;
//   * the token operand is loaded straight from L2 into mma.sync B fragments:
//     each lane reads 8 consecutive k of one token (16 B of bf16) and the
//     A fragment takes the same 8 k of a weight row from shared memory, so the
//     k order inside a 32-k step is a permutation shared by A and B (the dot
//     product is unchanged).
//
// Results are deterministic (fixed-order reductions everywhere). Numerics follow
// the reference model (oracle/ restatement): fp32 accumulation of bf16 products,
// residual stream fp32, x = bf16(h / rms(h)).
#include <type_traits>

#include "kernels.cuh"
#include "ptx.cuh"

namespace spin {
namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void mma16816(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

// Rows of unit u: half 0 = rows [row0, row0 + 8*MT), half 1 = rows [row1, row1 + 8*MT);
// m16 tile m takes rows 8m..8m+7 of each half as its rows 0-7 / 8-15.
__host__ __device__ __forceinline__ void unit_rows(int mode, int n_out, int hd, int MT, int u, int& row0, int& row1) {
  if (mode == kDpQkv) {  // half 1 = the RoPE partners (+head_dim/2) of half 0
    const int D = n_out / 3, per_sec = D / 16, per_head = hd / 16;
    const int sec = u / per_sec, j = u % per_sec;
    row0 = sec * D + (j / per_head) * hd + (j % per_head) * 8;
    row1 = row0 + hd / 2;
  } else if (mode == kDpGateUp) {  // half 1 = the up rows of half 0's gate rows
    row0 = 8 * MT * u;
    row1 = n_out / 2 + row0;
  } else {
    row0 = 16 * u;
    row1 = row0 + 8;
  }
}

__host__ __device__ __forceinline__ int unit_mt(int mode, int n_out) {
  return mode == kDpGateUp && (n_out / 2) % 16 == 0 ? 2 : 1;
}

// Slab layout: unit u's weights are one contiguous block [kb][half][8*MT rows][64 k] =
// exactly its shared-memory image (rows keep the 128-B swizzle of the tiled layout,
// chunk c of row r at c ^ (r % 8)), so a CTA fetches its whole unit with a few 16-KB
// bulk copies (1-KB row-group copies out of the tiled layout are request-bound: the
// draft GEMMs streamed at ~1.3 TB/s that way).
__global__ void slab_weights_kernel(const bf16* __restrict__ tiled, bf16* __restrict__ slab, int mode, int n_out,
                                    int K, int hd) {
  const int KB = (K + 63) / 64, MT = unit_mt(mode, n_out);
  const int64_t per_unit = static_cast<int64_t>(KB) * 2 * MT * 8 * 8;  // 16-B chunks
  const int64_t total = static_cast<int64_t>(n_out / (16 * MT)) * per_unit;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int u = static_cast<int>(e / per_unit);
    int64_t r_ = e % per_unit;
    const int pc = static_cast<int>(r_ % 8);
    r_ /= 8;
    const int j = static_cast<int>(r_ % (8 * MT));
    r_ /= 8 * MT;
    const int h = static_cast<int>(r_ % 2), kb = static_cast<int>(r_ / 2);
    int row0, row1;
    unit_rows(mode, n_out, hd, MT, u, row0, row1);
    const int r = (h ? row1 : row0) + j;
    const uint4* src =
        reinterpret_cast<const uint4*>(tiled + (static_cast<size_t>(r >> 7) * KB + kb) * 8192 + (r & 127) * 64) + pc;
    reinterpret_cast<uint4*>(slab)[e] = *src;
  }
}

template <int NW, int NT, int MT, bool NORM>
struct DpCfg {
  static constexpr int kSlab = MT * 16 * 128;                  // bytes of one 64-k atom of the unit
  static constexpr int kXRegs = NT * 4;                        // registers per 32-k step of the token operand
  static constexpr int kBatch = kXRegs >= 64 ? 1 : 64 / kXRegs;  // 32-k steps loaded per round trip
  static constexpr int kRed = NW * MT * NT * 32 * 4;           // cross-warp reduction floats
  static constexpr int kAtomsPerCopy = 8 / MT;                 // 16-KB bulk copies
  __host__ __device__ static constexpr size_t inv_off(int KB) {
    return (static_cast<size_t>(KB) * kSlab + KB * 8 + 15) / 16 * 16;
  }
  static constexpr size_t smem_bytes(int KB) { return inv_off(KB) + NT * 8 * 4 + kRed * 4; }
};

template <int NW, int NT, int MT, bool NORM>
__global__ void __launch_bounds__(NW * 32, NW <= 8 ? 2 : 1) dproj_kernel(DraftProj a) {
  using C = DpCfg<NW, NT, MT, NORM>;
  extern __shared__ __align__(128) uint8_t smem[];
  const int K = a.K, KB = (K + 63) / 64, T = a.T;
  uint8_t* slab = smem;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(KB) * C::kSlab);
  float* inv_s = reinterpret_cast<float*>(smem + C::inv_off(KB));
  float* red = inv_s + NT * 8;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane >> 2, t4 = lane & 3;
  const int u = blockIdx.x;
  const bool stamp = a.st != nullptr && threadIdx.x == 0;
  if (stamp) a.st[4 * u] = ptx::globaltimer();
  int row0, row1;
  unit_rows(a.mode, a.n_out, a.g.head_dim, MT, u, row0, row1);

  // ---- weights first (never depend on the previous kernel): the unit's slab in 16-KB copies
  constexpr int APC = C::kAtomsPerCopy;
  if (threadIdx.x == 0) {
    const int n_copies = (KB + APC - 1) / APC;
    for (int c = 0; c < n_copies; ++c) ptx::mbar_init(&bar[c], 1);
    ptx::fence_mbar_init();
    const uint64_t pol = ptx::policy_evict_first();
    const uint8_t* src = reinterpret_cast<const uint8_t*>(a.w) + static_cast<size_t>(u) * KB * C::kSlab;
    for (int c = 0; c < n_copies; ++c) {
      const uint32_t bytes = static_cast<uint32_t>(min(APC, KB - c * APC)) * C::kSlab;
      ptx::mbar_arrive_expect_tx(&bar[c], bytes);
      ptx::bulk_load(slab + static_cast<size_t>(c) * APC * C::kSlab, src + static_cast<size_t>(c) * APC * C::kSlab,
                     bytes, &bar[c], pol);
    }
  }
  // ---- epilogue operands that are final before this grid starts (the forward's row
  // metadata, RoPE tables, and the residual h, last written two or more kernels back;
  // each kernel of the chain triggers its dependents only after its own wait)
  const int tA = (warp % NT) * 8 + 2 * t4;  // epilogue warps (m, nt) = (warp / NT, warp % NT)
  const bool epi = warp < MT * NT;
  float pre[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
  int pre_pos[2] = {0, 0}, pre_slot[2] = {-1, -1};
  if (epi) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int tt = tA + e;
      if (tt >= T) continue;
      if (a.mode == kDpQkv) {
        pre_pos[e] = a.row_pos[tt];
        pre_slot[e] = a.row_slot[tt];
      } else if (a.mode == kDpResid) {
        pre[e][0] = __ldcg(a.h + static_cast<size_t>(tt) * a.n_out + row0 + g);
        pre[e][1] = __ldcg(a.h + static_cast<size_t>(tt) * a.n_out + row1 + g);
      }
    }
    if (a.mode == kDpQkv) {
      const int D = a.g.n_heads * a.g.head_dim, half = a.g.head_dim / 2, i = (row0 % D + g) % a.g.head_dim;
#pragma unroll
      for (int e = 0; e < 2; ++e)
        if (tA + e < T) {
          pre[e][0] = a.rcos[static_cast<size_t>(pre_pos[e]) * half + i];
          pre[e][1] = a.rsin[static_cast<size_t>(pre_pos[e]) * half + i];
        }
    }
  }
  __syncthreads();
  ptx::grid_dep_wait();
  // dependents may launch now: their prologues only read weights and data that is final
  // once this grid's own dependency wait has returned
  ptx::grid_dep_launch();
  if (stamp) a.st[4 * u + 1] = ptx::globaltimer();

  // ---- this warp's 32-k steps: atoms warp, warp + NW, ...; two steps per atom
  const int n_steps = warp < KB ? 2 * ((KB - warp + NW - 1) / NW) : 0;
  // token operand: bf16 rows (the residual producers keep a bf16 copy of h beside the
  // fp32 stream, so the norm consumers load 16 B per 8 k like the others)
  uint4 xr[C::kBatch][NT];
  auto load_batch = [&](int s0) {
#pragma unroll
    for (int b = 0; b < C::kBatch; ++b) {
      const int s = s0 + b;
      const int kb = warp + NW * (s >> 1);
      const int kk = kb * 64 + (s & 1) * 32 + t4 * 8;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int tok = nt * 8 + g;
        const bool ok = s < n_steps && tok < T && kk < K;
        xr[b][nt] = ok ? __ldcg(reinterpret_cast<const uint4*>(a.x + static_cast<size_t>(tok) * K + kk))
                       : make_uint4(0u, 0u, 0u, 0u);
      }
    }
  };
  load_batch(0);
  if constexpr (NORM) {
    // 1 / rms of every token from the producers' per-unit sums of squares (fixed order);
    // all of a warp's loads are in flight together (n_ssp <= 4 x 32)
    constexpr int TPW = (NT * 8 + NW - 1) / NW;  // tokens per warp
    float ss[TPW][4];
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int t = warp + NW * j;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int v = lane + 32 * r;
        ss[j][r] = (t < T && v < a.n_ssp) ? __ldcg(a.ssp + static_cast<size_t>(t) * a.n_ssp + v) : 0.f;
      }
    }
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      float x = (ss[j][0] + ss[j][1]) + (ss[j][2] + ss[j][3]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
      const int t = warp + NW * j;
      if (lane == 0 && t < NT * 8)
        inv_s[t] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(x, static_cast<float>(K)), a.eps)));
    }
  }
  // (inv_s is published by the barrier before the cross-warp reduction: the RMSNorm
  // scale is a per-token factor, applied to the reduced outputs, so the weight and
  // token loads never wait on the sums of squares)

  float acc[MT][NT][4];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[m][nt][0] = acc[m][nt][1] = acc[m][nt][2] = acc[m][nt][3] = 0.f;

  const uint32_t slab_u = ptx::smem_u32(slab);
  for (int s0 = 0; s0 < n_steps; s0 += C::kBatch) {
    if (s0 > 0) load_batch(s0);
#pragma unroll
    for (int b = 0; b < C::kBatch; ++b) {
      const int s = s0 + b;
      if (s >= n_steps) break;
      const int kb = warp + NW * (s >> 1);
      if ((s & 1) == 0) ptx::mbar_wait(&bar[kb / APC], 0);
      const uint32_t chunk = static_cast<uint32_t>(((s & 1) * 4 + t4) ^ g) << 4;
      uint4 wa[MT], wb[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const uint32_t base = slab_u + kb * C::kSlab + (8 * m + g) * 128 + chunk;
        wa[m] = lds128(base);
        wb[m] = lds128(base + MT * 1024);
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const uint4 x = xr[b][nt];
        const uint32_t b0 = x.x, b1 = x.y, b2 = x.z, b3 = x.w;
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          mma16816(acc[m][nt], wa[m].x, wb[m].x, wa[m].y, wb[m].y, b0, b1);
          mma16816(acc[m][nt], wa[m].z, wb[m].z, wa[m].w, wb[m].w, b2, b3);
        }
      }
    }
  }
  if (stamp) a.st[4 * u + 2] = ptx::globaltimer();

  // ---- fixed-order cross-warp reduction; warp (m, nt) finishes tile m x n-tile nt
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
      *reinterpret_cast<float4*>(red + (((warp * MT + m) * NT + nt) * 32 + lane) * 4) =
          make_float4(acc[m][nt][0], acc[m][nt][1], acc[m][nt][2], acc[m][nt][3]);
  __syncthreads();
  if (!epi) return;
  const int m = warp / NT, nt = warp % NT;
  float c[4] = {0.f, 0.f, 0.f, 0.f};
  const int nw_used = min(NW, KB);
  for (int w = 0; w < nw_used; ++w) {
    const float4 v = *reinterpret_cast<const float4*>(red + (((w * MT + m) * NT + nt) * 32 + lane) * 4);
    c[0] += v.x, c[1] += v.y, c[2] += v.z, c[3] += v.w;
  }
  // c[0], c[1]: half-0 row (row0 + 8m + g), tokens tA, tA + 1; c[2], c[3]: half-1 row, same tokens
  if constexpr (NORM) {
    const float i0 = inv_s[tA], i1 = inv_s[tA + 1];
    c[0] = __fmul_rn(c[0], i0), c[2] = __fmul_rn(c[2], i0);
    c[1] = __fmul_rn(c[1], i1), c[3] = __fmul_rn(c[3], i1);
  }
  if (a.mode == kDpQkv) {
    const AttnGeom& G = a.g;
    const int D = G.n_heads * G.head_dim, hd = G.head_dim, half = hd / 2;
    const int sec = row0 / D, f0 = row0 % D + g, hh = f0 / hd, i = f0 % hd;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int tt = tA + e;
      if (tt >= T) continue;
      const float x0 = c[e], x1 = c[2 + e];
      const int pos = pre_pos[e], slot = pre_slot[e];
      if (sec == 2) {
        if (slot < 0) continue;
        const size_t kv = ((((static_cast<size_t>(G.layer) * G.slots + slot) * G.n_heads + hh) * G.ctx) + pos) * hd;
        G.v_cache[kv + kv_swz(pos, i)] = __float2bfloat16_rn(x0);
        G.v_cache[kv + kv_swz(pos, i + half)] = __float2bfloat16_rn(x1);
        continue;
      }
      const float cs = pre[e][0], sn = pre[e][1];
      const float y0 = __fsub_rn(__fmul_rn(x0, cs), __fmul_rn(x1, sn));
      const float y1 = __fadd_rn(__fmul_rn(x1, cs), __fmul_rn(x0, sn));
      if (sec == 0) {
        a.q[static_cast<size_t>(tt) * D + f0] = y0;
        a.q[static_cast<size_t>(tt) * D + f0 + half] = y1;
      } else {
        if (slot < 0) continue;
        const size_t kv = ((((static_cast<size_t>(G.layer) * G.slots + slot) * G.n_heads + hh) * G.ctx) + pos) * hd;
        G.k_cache[kv + kv_swz(pos, i)] = __float2bfloat16_rn(y0);
        G.k_cache[kv + kv_swz(pos, i + half)] = __float2bfloat16_rn(y1);
      }
    }
  } else if (a.mode == kDpGateUp) {
    const int F = a.n_out / 2, f = row0 + 8 * m + g;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int tt = tA + e;
      if (tt >= T) continue;
      const float gt = c[e], up = c[2 + e];
      a.act[static_cast<size_t>(tt) * F + f] =
          __float2bfloat16_rn(__fmul_rn(__fdiv_rn(gt, __fadd_rn(1.0f, expf(-gt))), up));
    }
  } else {  // residual: h += y, and this unit's sum of squares per token
    const int D = a.n_out, n0 = row0 + g, n1 = row1 + g;
    float ss[2] = {0.f, 0.f};
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int tt = tA + e;
      if (tt >= T) continue;
      float* hr = a.h + static_cast<size_t>(tt) * D;
      const float h0 = __fadd_rn(pre[e][0], c[e]), h1 = __fadd_rn(pre[e][1], c[2 + e]);
      hr[n0] = h0;
      hr[n1] = h1;
      a.hb[static_cast<size_t>(tt) * D + n0] = __float2bfloat16_rn(h0);
      a.hb[static_cast<size_t>(tt) * D + n1] = __float2bfloat16_rn(h1);
      ss[e] = __fadd_rn(__fmul_rn(h0, h0), __fmul_rn(h1, h1));
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      ss[0] += __shfl_xor_sync(kFull, ss[0], o);
      ss[1] += __shfl_xor_sync(kFull, ss[1], o);
    }
    if (g == 0) {
      if (tA < T) a.ssp_out[static_cast<size_t>(tA) * (a.n_out / 16) + u] = ss[0];
      if (tA + 1 < T) a.ssp_out[static_cast<size_t>(tA + 1) * (a.n_out / 16) + u] = ss[1];
    }
  }
  if (stamp) a.st[4 * u + 3] = ptx::globaltimer();
}

// h = embedding rows (fp32), ssp[0][t] = sum of squares (one unit).
__global__ void __launch_bounds__(256) embed_ss_kernel(const bf16* __restrict__ emb, const int32_t* __restrict__ tok,
                                                       int T, int D, float* __restrict__ h, bf16* __restrict__ hb,
                                                       float* __restrict__ ssp) {
  __shared__ float red[32];
  ptx::grid_dep_wait();
  ptx::grid_dep_launch();
  const int t = blockIdx.x;
  const bf16* e = emb + static_cast<size_t>(tok[t]) * D;
  float ss = 0.f;
  for (int i = 2 * threadIdx.x; i < D; i += 2 * blockDim.x) {
    const __nv_bfloat162 raw = *reinterpret_cast<const __nv_bfloat162*>(e + i);
    const float2 v = __bfloat1622float2(raw);
    *reinterpret_cast<float2*>(h + static_cast<size_t>(t) * D + i) = v;
    *reinterpret_cast<__nv_bfloat162*>(hb + static_cast<size_t>(t) * D + i) = raw;
    ss += v.x * v.x + v.y * v.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(kFull, ss, o);
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    float tot = 0.f;
    for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) tot += red[w];
    ssp[t] = tot;
  }
}

// xn = bf16(h / rms(h)) with rms from the per-unit sums of squares (the lm_head input).
__global__ void __launch_bounds__(256) norm_ss_kernel(const float* __restrict__ h, const float* __restrict__ ssp,
                                                      int n_ssp, int T, int D, float eps, bf16* __restrict__ xn) {
  __shared__ float inv_s;
  ptx::grid_dep_wait();
  ptx::grid_dep_launch();
  const int t = blockIdx.x;
  if (threadIdx.x < 32) {
    float ss = 0.f;
    for (int v = threadIdx.x; v < n_ssp; v += 32) ss += ssp[static_cast<size_t>(t) * n_ssp + v];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(kFull, ss, o);
    if (threadIdx.x == 0)
      inv_s = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(ss, static_cast<float>(D)), eps)));
  }
  __syncthreads();
  const float inv = inv_s;
  for (int i = 4 * threadIdx.x; i < D; i += 4 * blockDim.x) {
    const float4 v = *reinterpret_cast<const float4*>(h + static_cast<size_t>(t) * D + i);
    uint2 o;
    o.x = pack_bf16(__fmul_rn(v.x, inv), __fmul_rn(v.y, inv));
    o.y = pack_bf16(__fmul_rn(v.z, inv), __fmul_rn(v.w, inv));
    *reinterpret_cast<uint2*>(xn + static_cast<size_t>(t) * D + i) = o;
  }
}

template <typename K, typename... Args>
cudaError_t launch_pdl(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_allowed();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <int NW, int NT, int MT, bool NORM>
cudaError_t launch_t(const DraftProj& a, int units, cudaStream_t s) {
  using C = DpCfg<NW, NT, MT, NORM>;
  const int KB = (a.K + 63) / 64;
  const size_t smem = C::smem_bytes(KB);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  ensure_smem_optin(reinterpret_cast<const void*>(dproj_kernel<NW, NT, MT, NORM>), smem);
  return launch_pdl(dproj_kernel<NW, NT, MT, NORM>, dim3(units), dim3(NW * 32), smem, s, a);
}

template <int NT, int MT, bool NORM>
cudaError_t launch_nw(const DraftProj& a, int units, cudaStream_t s) {
  // many 64-k atoms (the down projection) and few units: more warps per CTA
  return (a.K > 1024) ? launch_t<16, NT, MT, NORM>(a, units, s) : launch_t<8, NT, MT, NORM>(a, units, s);
}

template <int MT, bool NORM>
cudaError_t launch_nt(const DraftProj& a, int units, cudaStream_t s) {
  const int nt = (a.T + 7) / 8;
  if (nt <= 1) return launch_nw<1, MT, NORM>(a, units, s);
  if (nt <= 2) return launch_nw<2, MT, NORM>(a, units, s);
  return launch_nw<4, MT, NORM>(a, units, s);
}

}  // namespace

bool draft_fused_supported(int D, int H, int hd, int F, int T) {
  return T >= 1 && T <= kDraftMaxT && D % 64 == 0 && hd % 16 == 0 && H * hd == D && F % 8 == 0 &&
         F <= 8192 && D <= 2048;  // n_ssp = D / 16 <= 128 (dproj inv loads)
}

int draft_proj_units(const DraftProj& a) { return a.n_out / (16 * unit_mt(a.mode, a.n_out)); }

size_t draft_slab_elems(int n_out, int K) { return static_cast<size_t>(n_out) * ((K + 63) / 64) * 64; }

void launch_slab_weights(const bf16* tiled, bf16* slab, int mode, int n_out, int K, int hd, cudaStream_t s) {
  slab_weights_kernel<<<1184, 256, 0, s>>>(tiled, slab, mode, n_out, K, hd);
}

cudaError_t launch_draft_proj(const DraftProj& a, cudaStream_t s) {
  switch (a.mode) {
    case kDpQkv:
      return launch_nt<1, true>(a, a.n_out / 16, s);
    case kDpGateUp: {
      const int F = a.n_out / 2;
      return F % 16 == 0 ? launch_nt<2, true>(a, F / 16, s) : launch_nt<1, true>(a, F / 8, s);
    }
    default:
      return launch_nt<1, false>(a, a.n_out / 16, s);
  }
}

void launch_embed_ss(const bf16* emb, const FwdMeta& m, int T, int D, float* h, bf16* hb, float* ssp,
                     cudaStream_t s) {
  launch_pdl(embed_ss_kernel, dim3(T), dim3(256), 0, s, emb, static_cast<const int32_t*>(m.row_tok), T, D, h, hb, ssp);
}

void launch_norm_ss(const float* h, const float* ssp, int n_ssp, int T, int D, float eps, bf16* xn, cudaStream_t s) {
  launch_pdl(norm_ss_kernel, dim3(T), dim3(256), 0, s, h, ssp, n_ssp, T, D, eps, xn);
}

}  // namespace spin
