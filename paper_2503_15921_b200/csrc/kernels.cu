// Memory-bound kernels: per-forward metadata + device request decomposition,
// embedding/RMSNorm, split-K reductions fused with RoPE + KV append, residual +
// RMSNorm and SwiGLU, greedy acceptance with KV rollback, synthetic weights,
// and the fp64 toy-mode packed attention operator.
#include <algorithm>
#include <cstdio>

#include "kernels.cuh"
#include "ptx.cuh"

namespace spin {

namespace {

constexpr unsigned kFull = 0xffffffffu;

// Fixed-order sum of the stream-K partial slots of 4 consecutive features
// (slot 0..np-1, deterministic); np comes from the plan's host-built piece table.
// The first kUnrollPieces partial loads are predicated rather than looped so that a
// caller summing several groups has all of their loads in flight at once.
constexpr int kUnrollPieces = 2;

// SPIN_STAMPS: per-block globaltimer stamps (start, dependency released, -, end) of the
// epilogue kernels of target layer 1 (engine.cu stamp_slot kinds 16-18)
__device__ __forceinline__ void stamp(unsigned long long* st, int j) {
  if (st != nullptr && threadIdx.x == 0) st[4 * (blockIdx.y * gridDim.x + blockIdx.x) + j] = ptx::globaltimer();
}
__device__ __forceinline__ float4 sum_pieces4(const float* __restrict__ part, const PieceMap& pm, int T, int n_out,
                                              int t, int n) {
  const int np = pm.tile_pieces(t, n);
  const size_t stride = static_cast<size_t>(T) * n_out;
  const float* p = part + static_cast<size_t>(t) * n_out + n;
  float4 v[kUnrollPieces];
#pragma unroll
  for (int s = 0; s < kUnrollPieces; ++s)
    if (s < np) v[s] = __ldg(reinterpret_cast<const float4*>(p + s * stride));
  float4 acc = v[0];
#pragma unroll
  for (int s = 1; s < kUnrollPieces; ++s)
    if (s < np) {
      acc.x = __fadd_rn(acc.x, v[s].x);
      acc.y = __fadd_rn(acc.y, v[s].y);
      acc.z = __fadd_rn(acc.z, v[s].z);
      acc.w = __fadd_rn(acc.w, v[s].w);
    }
  for (int s = kUnrollPieces; s < np; ++s) {
    const float4 w = __ldg(reinterpret_cast<const float4*>(p + s * stride));
    acc.x = __fadd_rn(acc.x, w.x);
    acc.y = __fadd_rn(acc.y, w.y);
    acc.z = __fadd_rn(acc.z, w.z);
    acc.w = __fadd_rn(acc.w, w.w);
  }
  return acc;
}

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}

// sum_pieces4 split in two so that a kernel looks its piece counts up BEFORE the PDL
// dependency wait (the table is constant) and issues every slot load right after it:
// set() (pre-wait), issue() (post-wait), sum() -- same fixed slot order as sum_pieces4.
struct Pieces4 {
  const float* p;
  int np;
  float4 v[kUnrollPieces];
  __device__ __forceinline__ void set(const float* part, const PieceMap& pm, int T, int n_out, int t, int n) {
    np = pm.tile_pieces(t, n);
    p = part + static_cast<size_t>(t) * n_out + n;
  }
  __device__ __forceinline__ void issue(size_t stride) {
#pragma unroll
    for (int s = 0; s < kUnrollPieces; ++s)
      if (s < np) v[s] = __ldg(reinterpret_cast<const float4*>(p + s * stride));
  }
  __device__ __forceinline__ float4 sum(size_t stride) const {
    float4 acc = v[0];
#pragma unroll
    for (int s = 1; s < kUnrollPieces; ++s)
      if (s < np) acc = add4(acc, v[s]);
    for (int s = kUnrollPieces; s < np; ++s) acc = add4(acc, __ldg(reinterpret_cast<const float4*>(p + s * stride)));
    return acc;
  }
};

// SMs of the current device (grid sizing of the one-wave epilogue kernels).
int device_sms() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n;
  }
  return cache[dev];
}

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32, nw = blockDim.x / 32;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < nw; ++i) t += red[i];
  return t;
}

__device__ __forceinline__ void amax_better(float& v, int& i, float ov, int oi) {
  if (ov > v || (ov == v && oi < i)) {
    v = ov;
    i = oi;
  }
}

// Token id of the argmax over all lm_head tiles for one row (lowest index on ties).
__device__ int row_argmax_warp(const float* val, const int32_t* idx, int tiles, int T, int row) {
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int tl = threadIdx.x % 32; tl < tiles; tl += 32)
    amax_better(bv, bi, val[static_cast<size_t>(tl) * T + row], idx[static_cast<size_t>(tl) * T + row]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(kFull, bv, o);
    const int oi = __shfl_xor_sync(kFull, bi, o);
    amax_better(bv, bi, ov, oi);
  }
  return bi;
}

// ------------------------------------------------------------------ meta
constexpr int kMetaThreads = 512;
constexpr int kMaxReq = 1024;
constexpr int kMaxSeg = 2 * kMaxReq;
constexpr size_t kMetaSmem = (11 * kMaxReq + 12 + 6 * kMaxSeg) * sizeof(int);

__global__ void __launch_bounds__(kMetaThreads) meta_kernel(MetaArgs a, SlotState st, FwdMeta m) {
  extern __shared__ int msm[];
  int* s_len = msm;                   // [n] kv length per request
  int* s_order = s_len + kMaxReq;     // [n] requests by decreasing length
  int* s_used = s_order + kMaxReq;    // [rows] fill, later row counts
  int* s_ptr = s_used + kMaxReq;      // [rows + 1] CSR
  int* s_misc = s_ptr + kMaxReq + 4;  // [0] nseg
  int* s_rlen = s_misc + kMaxReq;     // [rows] attention pieces per row
  int* s_rs0 = s_rlen + kMaxReq;      // [n] first segment of each request
  int* s_rns = s_rs0 + kMaxReq;       // [n] its segment count
  int* s_np = s_rns + kMaxReq;        // [n] attention pieces per request
  int* s_rbase = s_np + kMaxReq;      // [rows + 1] first piece of each row
  int* s_rptr = s_rbase + kMaxReq + 4;  // [n + 1] first merge-list entry of each request
  int* s_pofs = s_rptr + kMaxReq + 4;   // [nseg] first piece of each segment within its request
  int* s_seg = s_pofs + kMaxSeg;        // [nseg][5]
  const int n = a.n_req;
  const int tid = threadIdx.x;
  const int warp = tid / 32, lane = tid % 32;
  const int W = st.window;

  ptx::grid_dep_wait();
  ptx::grid_dep_launch();  // the next kernel's prologue reads nothing of ours before its wait
  // ---- collect the previous draft step's argmax (one warp per request)
  if (a.mode == kMetaDraftK || a.mode == kMetaCollect) {
    for (int r = warp; r < n; r += kMetaThreads / 32) {
      const int row = r * a.prev_qlen + a.prev_qlen - 1;
      int tok = row_argmax_warp(a.amax_val, a.amax_idx, a.amax_tiles, a.prev_t, row);
      if (tok < 0 || tok >= a.amax_tiles * 128) {  // all-NaN logits: report (status 3), never index with it
        if (lane == 0 && m.err && atomicCAS(m.err, 0, 3) == 0) {
          m.err[1] = a.list[r], m.err[2] = a.ssm, m.err[3] = a.step, m.err[4] = row;
          __threadfence_system();
        }
        tok = 0;
      }
      if (lane == 0) st.drafts[static_cast<size_t>(a.list[r]) * W + a.step - 1] = tok;
    }
    __syncthreads();
  }
  if (a.mode == kMetaCollect) {
    for (int r = tid; r < n; r += kMetaThreads) {
      const int slot = a.list[r];
      st.ssm_len[static_cast<size_t>(a.ssm) * st.slots + slot] = st.committed[slot] + W - 1;
    }
    return;
  }
  // ---- rows and requests
  for (int r = tid; r < n; r += kMetaThreads) {
    if (a.mode == kMetaExtend) {
      s_len[r] = m.req_kvlen[r];
      continue;
    }
    const int slot = a.list[r];
    const int c = st.committed[slot];
    const int32_t* hist = st.tokens + static_cast<size_t>(slot) * st.ctx;
    const int32_t* dr = st.drafts + static_cast<size_t>(slot) * W;
    int ql, kv;
    if (a.mode == kMetaVerify) {
      ql = W + 1;
      kv = c + W;
      const int q0 = r * ql;
      for (int j = 0; j < ql; ++j) {
        m.row_tok[q0 + j] = j == 0 ? hist[c - 1] : dr[j - 1];
        m.row_slot[q0 + j] = slot;
        m.row_pos[q0 + j] = c - 1 + j;
      }
    } else if (a.mode == kMetaDraft0) {
      ql = 2;
      kv = c;
      for (int j = 0; j < 2; ++j) {
        m.row_tok[2 * r + j] = hist[c - 2 + j];
        m.row_slot[2 * r + j] = slot;
        m.row_pos[2 * r + j] = c - 2 + j;
      }
    } else {  // DraftK
      ql = 1;
      kv = c + a.step;
      m.row_tok[r] = dr[a.step - 1];
      m.row_slot[r] = slot;
      m.row_pos[r] = c - 1 + a.step;
    }
    m.req_slot[r] = slot;
    m.req_qstart[r] = r * ql;
    m.req_qlen[r] = ql;
    m.req_kvlen[r] = kv;
    s_len[r] = kv;
  }
  __syncthreads();

  // ---- request decomposition (packing.cpp:16-103, restated for one warp)
  const int rows = a.padded ? n : min(a.width > 0 ? a.width : n, n);
  if (!a.padded) {
    for (int i = tid; i < n; i += kMetaThreads) {  // stable rank by decreasing length
      const int li = s_len[i];
      int rank = 0;
      for (int j = 0; j < n; ++j) rank += (s_len[j] > li) || (s_len[j] == li && j < i);
      s_order[rank] = i;
    }
    for (int r = tid; r < rows; r += kMetaThreads) s_used[r] = 0;
  }
  __syncthreads();
  if (warp == 0) {
    int nseg = 0;
    if (a.padded) {
      int longest = 0;
      for (int i = lane; i < n; i += 32) longest = max(longest, s_len[i]);
      for (int o = 16; o > 0; o >>= 1) longest = max(longest, __shfl_xor_sync(kFull, longest, o));
      for (int i = lane; i < n; i += 32) {
        int* sg = s_seg + 5 * i;
        sg[0] = i, sg[1] = i, sg[2] = 0, sg[3] = longest, sg[4] = 0;
      }
      nseg = n;
      if (lane == 0) s_misc[2] = longest;
    } else {
      long long total = 0;
      for (int i = lane; i < n; i += 32) total += s_len[i];
      for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(kFull, total, o);
      // With splitting allowed the first candidate L = ceil(total / rows)
      // always fits (capacity >= total), so the reference's upward search
      // stops at its first iteration.
      const int L = static_cast<int>((total + rows - 1) / rows);
      if (lane == 0) s_misc[2] = L;
      for (int k = 0; k < n; ++k) {
        const int id = s_order[k];
        const int need = s_len[id];
        int home = -1;
        for (int base = 0; base < rows && home < 0; base += 32) {
          const int r = base + lane;
          const unsigned mask = __ballot_sync(kFull, r < rows && L - s_used[r] >= need);
          if (mask) home = base + __ffs(mask) - 1;
        }
        if (home >= 0) {
          if (lane == 0) {
            int* sg = s_seg + 5 * nseg;
            sg[0] = id, sg[1] = home, sg[2] = s_used[home], sg[3] = s_used[home] + need, sg[4] = 0;
            s_used[home] += need;
          }
          ++nseg;
          __syncwarp();
          continue;
        }
        int remaining = need, done = 0;
        for (int base = 0; base < rows && remaining > 0; base += 32) {
          const int r = base + lane;
          const int room = r < rows ? max(0, L - s_used[r]) : 0;
          int incl = room;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
          }
          const int excl = incl - room;
          const int take = min(room, max(0, remaining - excl));
          const unsigned mask = __ballot_sync(kFull, take > 0);
          if (take > 0) {
            int* sg = s_seg + 5 * (nseg + __popc(mask & ((1u << lane) - 1u)));
            sg[0] = id, sg[1] = r, sg[2] = s_used[r], sg[3] = s_used[r] + take, sg[4] = done + excl;
            s_used[r] += take;
          }
          nseg += __popc(mask);
          const int chunk = __shfl_sync(kFull, incl, 31);
          const int taken = min(remaining, chunk);
          remaining -= taken;
          done += taken;
          __syncwarp();
        }
      }
    }
    if (lane == 0) s_misc[0] = nseg;
  }
  __syncthreads();
  const int nseg = s_misc[0];
  const int nch = max(1, a.chunks);
  // ---- segments out; per-request segment ranges (a request's segments are consecutive)
  if (tid == 0) {
    s_misc[1] = 0;
    m.n_seg[0] = nseg;
    m.n_seg[1] = s_misc[2];
  }
  __syncthreads();
  for (int s = tid; s < nseg; s += kMetaThreads) {
#pragma unroll
    for (int e = 0; e < 5; ++e) m.seg[5 * s + e] = s_seg[5 * s + e];
    const int rq = s_seg[5 * s];
    if (s == 0 || s_seg[5 * (s - 1)] != rq) {
      int e = s + 1;
      while (e < nseg && s_seg[5 * e] == rq) ++e;
      m.req_seg0[rq] = s;
      m.req_nseg[rq] = e - s;
      s_rs0[rq] = s;
      s_rns[rq] = e - s;
    }
    atomicMax(&s_misc[1], s_seg[5 * s + 3]);
  }
  __syncthreads();
  // Attention work items: every pack row is cut into nch chunks of C columns;
  // a piece = one segment's part inside one chunk (the split-KV unit).
  const int C = max(16, ((s_misc[1] + nch - 1) / nch + 15) / 16 * 16);
  auto touched = [&](const int* sg) { return (sg[3] - 1) / C - sg[2] / C + 1; };
  // ---- per pack row: segment count, used length, pieces
  for (int r = tid; r < rows; r += kMetaThreads) {
    int c = 0, len = 0, pcs = 0;
    for (int s = 0; s < nseg; ++s) {
      const int* sg = s_seg + 5 * s;
      if (sg[1] != r) continue;
      ++c;
      len = max(len, sg[3]);
      pcs += touched(sg);
    }
    s_used[r] = c;
    s_rlen[r] = pcs;
    m.row_len[r] = len;
  }
  // ---- per request: pieces and each segment's first piece index (token order)
  for (int rq = tid; rq < n; rq += kMetaThreads) {
    int run = 0;
    for (int s = s_rs0[rq]; s < s_rs0[rq] + s_rns[rq]; ++s) {
      s_pofs[s] = run;
      run += touched(s_seg + 5 * s);
    }
    s_np[rq] = run;
  }
  __syncthreads();
  // ---- exclusive scans: warp 0 row segments, warp 1 row pieces, warp 2 request pieces
  if (warp < 3) {
    const int* src = warp == 0 ? s_used : warp == 1 ? s_rlen : s_np;
    int* dst = warp == 0 ? s_ptr : warp == 1 ? s_rbase : s_rptr;
    const int cnt = warp == 2 ? n : rows;
    int carry = 0;
    for (int base = 0; base < cnt; base += 32) {
      const int r = base + lane;
      const int v = r < cnt ? src[r] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      if (r < cnt) dst[r] = carry + incl - v;
      carry += __shfl_sync(kFull, incl, 31);
    }
    if (lane == 0) dst[cnt] = carry;
  }
  __syncthreads();
  if (s_rbase[rows] > m.piece_cap) {  // piece buffers sized by the engine: flag, leave no work
    for (int r = tid; r <= rows * nch; r += kMetaThreads) m.item_ptr[r] = 0;
    for (int r = tid; r <= n; r += kMetaThreads) m.req_pptr[r] = 0;
    if (tid == 0) {
      m.n_pieces[0] = 0;
      if (m.err) *reinterpret_cast<volatile int32_t*>(m.err) = 1;  // may be host-mapped
    }
    return;
  }
  for (int r = tid; r <= rows; r += kMetaThreads) m.row_ptr[r] = s_ptr[r];
  for (int r = tid; r <= n; r += kMetaThreads) m.req_pptr[r] = s_rptr[r];
  if (tid == 0) {
    m.item_ptr[rows * nch] = s_rbase[rows];
    m.n_pieces[0] = s_rbase[rows];
  }
  // ---- placement (thread per row): pieces in (chunk, column) order + per-request merge lists
  for (int r = tid; r < rows; r += kMetaThreads) {
    int pos = s_ptr[r];
    for (int s = 0; s < nseg; ++s)
      if (s_seg[5 * s + 1] == r) m.row_seg[pos++] = s;
    int pc = s_rbase[r];
    for (int c = 0; c < nch; ++c) {
      m.item_ptr[r * nch + c] = pc;
      const int x0 = c * C, x1 = (c + 1) * C;
      for (int k = s_ptr[r]; k < s_ptr[r + 1]; ++k) {
        const int s = m.row_seg[k];
        const int* sg = s_seg + 5 * s;
        const int a0 = max(sg[2], x0), a1 = min(sg[3], x1);
        if (a0 >= a1) continue;
        const int rq = sg[0];
        int4* rec = reinterpret_cast<int4*>(m.pieces + 16 * pc);
        rec[0] = make_int4(rq, m.req_slot[rq], sg[4] + (a0 - sg[2]), a1 - a0);
        rec[1] = make_int4(m.req_qstart[rq], m.req_qlen[rq], m.req_kvlen[rq], s_np[rq]);
        rec[2] = make_int4(s_rptr[rq], 0, 0, 0);
        m.req_plist[s_rptr[rq] + s_pofs[s] + (c - sg[2] / C)] = pc;
        ++pc;
      }
    }
  }
}

// ------------------------------------------------------------------ norms
constexpr int kRowThreads = 256;

// x = bf16(row * 1/sqrt(mean(row^2) + eps)); row staged in shared memory.
__device__ __forceinline__ void rmsnorm_row(const float* row, int D, float eps, bf16* xn, float* red) {
  float ss = 0.f;
  for (int i = threadIdx.x; i < D; i += blockDim.x) ss += row[i] * row[i];
  const float tot = block_sum(ss, red);
  const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(tot, static_cast<float>(D)), eps)));
  for (int i = 4 * threadIdx.x; i < D; i += 4 * blockDim.x) {
    const float4 v = *reinterpret_cast<const float4*>(row + i);
    __nv_bfloat162 a = __floats2bfloat162_rn(__fmul_rn(v.x, inv), __fmul_rn(v.y, inv));
    __nv_bfloat162 b = __floats2bfloat162_rn(__fmul_rn(v.z, inv), __fmul_rn(v.w, inv));
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(xn + i) = u;
  }
}

__global__ void __launch_bounds__(kRowThreads) embed_norm_kernel(const bf16* __restrict__ emb, const int32_t* tok,
                                                                 int D, float eps, float* h, bf16* xn) {
  extern __shared__ float s_row[];
  __shared__ float red[32];
  ptx::grid_dep_wait();
  ptx::grid_dep_launch();  // dependents (the next GEMM) may start their weight prefetch now
  const int t = blockIdx.x;
  const bf16* e = emb + static_cast<size_t>(tok[t]) * D;
  for (int i = threadIdx.x; i < D; i += kRowThreads) {
    const float v = __bfloat162float(e[i]);
    s_row[i] = v;
    h[static_cast<size_t>(t) * D + i] = v;
  }
  __syncthreads();
  rmsnorm_row(s_row, D, eps, xn + static_cast<size_t>(t) * D, red);
}

// h += sum of the stream-K partials; xn = bf16(rmsnorm(h)). Each thread owns NV float4
// groups of the row (D <= NV * 1024) and keeps them in registers; the loads of PB pieces
// for all groups are issued before any add or store, so the row costs
// ceil((max_pieces - 1) / PB) + 1 L2 round trips.
template <int NV, int PB>
__global__ void __launch_bounds__(kRowThreads, 2) resid_norm_kernel(const float* __restrict__ part, PieceMap pm, int T,
                                                                 int D, float eps, float* __restrict__ h,
                                                                 bf16* __restrict__ xn, unsigned long long* st) {
  __shared__ float red[32];
  stamp(st, 0);
  const int t = blockIdx.x;
  const size_t stride = static_cast<size_t>(T) * D;
  const float* prow = part + static_cast<size_t>(t) * D;
  float4* hrow = reinterpret_cast<float4*>(h + static_cast<size_t>(t) * D);
  float4 v[NV], y[NV];
  int np[NV];
  int maxp = 0;
  // Before the dependency wait: the piece counts (constant table) and the residual row
  // (last written by the previous residual kernel, two launches back: final once the
  // projection that precedes us has passed its own wait and triggered).
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int i = 4 * (threadIdx.x + k * kRowThreads);
    np[k] = i < D ? pm.tile_pieces(t, i) : 0;
    maxp = max(maxp, np[k]);
    if (i < D) v[k] = __ldcg(hrow + (i >> 2));
  }
  ptx::grid_dep_wait();
  ptx::grid_dep_launch();  // dependents (the next GEMM) may start their weight prefetch now
  stamp(st, 1);
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int i = 4 * (threadIdx.x + k * kRowThreads);
    if (i < D) y[k] = __ldg(reinterpret_cast<const float4*>(prow + i));
  }
  for (int s0 = 1; s0 < maxp; s0 += PB) {
    float4 z[PB][NV];
#pragma unroll
    for (int b = 0; b < PB; ++b)
#pragma unroll
      for (int k = 0; k < NV; ++k)
        if (s0 + b < np[k])
          z[b][k] = __ldg(reinterpret_cast<const float4*>(prow + (s0 + b) * stride + 4 * (threadIdx.x + k * kRowThreads)));
#pragma unroll
    for (int b = 0; b < PB; ++b)
#pragma unroll
      for (int k = 0; k < NV; ++k)
        if (s0 + b < np[k]) {
          y[k].x = __fadd_rn(y[k].x, z[b][k].x), y[k].y = __fadd_rn(y[k].y, z[b][k].y);
          y[k].z = __fadd_rn(y[k].z, z[b][k].z), y[k].w = __fadd_rn(y[k].w, z[b][k].w);
        }
  }
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    if (np[k] == 0) continue;
    v[k].x = __fadd_rn(v[k].x, y[k].x), v[k].y = __fadd_rn(v[k].y, y[k].y);
    v[k].z = __fadd_rn(v[k].z, y[k].z), v[k].w = __fadd_rn(v[k].w, y[k].w);
    hrow[threadIdx.x + k * kRowThreads] = v[k];
    ss += v[k].x * v[k].x + v[k].y * v[k].y + v[k].z * v[k].z + v[k].w * v[k].w;
  }
  const float tot = block_sum(ss, red);
  const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(tot, static_cast<float>(D)), eps)));
  bf16* xrow = xn + static_cast<size_t>(t) * D;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    if (np[k] == 0) continue;
    __nv_bfloat162 a = __floats2bfloat162_rn(__fmul_rn(v[k].x, inv), __fmul_rn(v[k].y, inv));
    __nv_bfloat162 b = __floats2bfloat162_rn(__fmul_rn(v[k].z, inv), __fmul_rn(v[k].w, inv));
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(xrow + 4 * (threadIdx.x + k * kRowThreads)) = u;
  }
  stamp(st, 3);
}

// SwiGLU of the gate|up split-K partials: one wave of 2 x SMs blocks (small enough that
// the next GEMM's CTA stays co-resident and prefetches its weights meanwhile), each thread
// kSwiG groups of 4 features per pass with every slot load of the pass in flight; the
// first pass's piece counts are looked up before the dependency wait.
constexpr int kSwiG = 2;
__device__ __forceinline__ void swiglu_store(float4 g, float4 u, bf16* dst) {
  const float gs[4] = {g.x, g.y, g.z, g.w}, us[4] = {u.x, u.y, u.z, u.w};
  float r[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) r[i] = __fmul_rn(__fdiv_rn(gs[i], __fadd_rn(1.0f, expf(-gs[i]))), us[i]);
  __nv_bfloat162 a = __floats2bfloat162_rn(r[0], r[1]), b = __floats2bfloat162_rn(r[2], r[3]);
  uint2 o;
  o.x = *reinterpret_cast<uint32_t*>(&a);
  o.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(dst) = o;
}

__global__ void __launch_bounds__(kRowThreads, 2) swiglu_kernel(const float* __restrict__ part, PieceMap pm, int T,
                                                                int F, bf16* act, unsigned long long* st) {
  stamp(st, 0);
  const int per_row = F / 4;
  const int items = T * per_row;
  const int nthr = gridDim.x * blockDim.x;
  const size_t stride = static_cast<size_t>(T) * 2 * F;
  Pieces4 g[kSwiG], u[kSwiG];
  int it0 = blockIdx.x * blockDim.x + threadIdx.x;
  auto set = [&](int base) {
#pragma unroll
    for (int k = 0; k < kSwiG; ++k) {
      const int it = base + k * nthr;
      const int t = it / per_row, f = 4 * (it % per_row);
      if (it < items) {
        g[k].set(part, pm, T, 2 * F, t, f);
        u[k].set(part, pm, T, 2 * F, t, F + f);
      } else {
        g[k].np = u[k].np = 0;
      }
    }
  };
  set(it0);
  ptx::grid_dep_wait();
  ptx::grid_dep_launch();  // dependents (the next GEMM) may start their weight prefetch now
  stamp(st, 1);
  for (; it0 < items; it0 += kSwiG * nthr) {
    if (it0 != static_cast<int>(blockIdx.x * blockDim.x + threadIdx.x)) set(it0);
#pragma unroll
    for (int k = 0; k < kSwiG; ++k) g[k].issue(stride), u[k].issue(stride);
#pragma unroll
    for (int k = 0; k < kSwiG; ++k) {
      const int it = it0 + k * nthr;
      if (it >= items) continue;
      const int t = it / per_row, f = 4 * (it % per_row);
      swiglu_store(g[k].sum(stride), u[k].sum(stride), act + static_cast<size_t>(t) * F + f);
    }
  }
  stamp(st, 3);
}

// Split-K reduce of the QKV partials + RoPE on q and k + KV append: items of 4 rotary pairs
// of one token (q, k, v sections: 12 partial float4 loads), grid-stride over one wave of
// 2 x SMs blocks; the first item's row metadata, RoPE factors and piece counts are read
// before the dependency wait.
struct QkvItem {
  int t, nq, hh, i, slot, pos;
  float4 c, s;
  Pieces4 pc[6];  // q lo, q hi, k lo, k hi, v lo, v hi
};

__global__ void __launch_bounds__(kRowThreads, 2) qkv_epilogue_kernel(const float* __restrict__ part, PieceMap pm,
                                                                   FwdMeta m, int T, AttnGeom g,
                                                                   const float* __restrict__ rcos,
                                                                   const float* __restrict__ rsin, float* q,
                                                                   unsigned long long* st) {
  stamp(st, 0);
  const int H = g.n_heads, hd = g.head_dim, half = hd / 2, D = H * hd, N = 3 * D;
  const int per_row = H * half / 4;
  const int items = T * per_row;
  const size_t stride = static_cast<size_t>(T) * N;
  QkvItem x;
  auto set = [&](int it) {
    x.t = it / per_row;
    const int p4 = 4 * (it % per_row);
    x.hh = p4 / half, x.i = p4 % half;
    x.nq = x.hh * hd + x.i;
    x.slot = m.row_slot[x.t], x.pos = m.row_pos[x.t];
    x.c = *reinterpret_cast<const float4*>(rcos + static_cast<size_t>(x.pos) * half + x.i);
    x.s = *reinterpret_cast<const float4*>(rsin + static_cast<size_t>(x.pos) * half + x.i);
#pragma unroll
    for (int j = 0; j < 6; ++j) x.pc[j].set(part, pm, T, N, x.t, (j >> 1) * D + x.nq + (j & 1) * half);
  };
  int it = blockIdx.x * blockDim.x + threadIdx.x;
  if (it < items) set(it);
  ptx::grid_dep_wait();
  ptx::grid_dep_launch();  // dependents (attention) may stage their work list now
  stamp(st, 1);
  for (bool first = true; it < items; it += gridDim.x * blockDim.x, first = false) {
    if (!first) set(it);
#pragma unroll
    for (int j = 0; j < 6; ++j) x.pc[j].issue(stride);
    const float4 q0 = x.pc[0].sum(stride), q1 = x.pc[1].sum(stride);
    const float4 k0 = x.pc[2].sum(stride), k1 = x.pc[3].sum(stride);
    const float4 v0 = x.pc[4].sum(stride), v1 = x.pc[5].sum(stride);
    const float qa[4] = {q0.x, q0.y, q0.z, q0.w}, qb[4] = {q1.x, q1.y, q1.z, q1.w};
    const float ka[4] = {k0.x, k0.y, k0.z, k0.w}, kb[4] = {k1.x, k1.y, k1.z, k1.w};
    const float cs[4] = {x.c.x, x.c.y, x.c.z, x.c.w}, sn[4] = {x.s.x, x.s.y, x.s.z, x.s.w};
    float qo0[4], qo1[4], ko0[4], ko1[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      qo0[e] = __fsub_rn(__fmul_rn(qa[e], cs[e]), __fmul_rn(qb[e], sn[e]));
      qo1[e] = __fadd_rn(__fmul_rn(qb[e], cs[e]), __fmul_rn(qa[e], sn[e]));
      ko0[e] = __fsub_rn(__fmul_rn(ka[e], cs[e]), __fmul_rn(kb[e], sn[e]));
      ko1[e] = __fadd_rn(__fmul_rn(kb[e], cs[e]), __fmul_rn(ka[e], sn[e]));
    }
    float* qo = q + static_cast<size_t>(x.t) * D + x.nq;
    *reinterpret_cast<float4*>(qo) = make_float4(qo0[0], qo0[1], qo0[2], qo0[3]);
    *reinterpret_cast<float4*>(qo + half) = make_float4(qo1[0], qo1[1], qo1[2], qo1[3]);
    if (x.slot >= 0) {
      const size_t kv = ((((static_cast<size_t>(g.layer) * g.slots + x.slot) * H + x.hh) * g.ctx) + x.pos) * hd;
      auto put4 = [](bf16* dst, float a, float b, float c2, float d) {
        __nv_bfloat162 u = __floats2bfloat162_rn(a, b), w = __floats2bfloat162_rn(c2, d);
        uint2 o;
        o.x = *reinterpret_cast<uint32_t*>(&u);
        o.y = *reinterpret_cast<uint32_t*>(&w);
        *reinterpret_cast<uint2*>(dst) = o;
      };
      // 4 consecutive dims stay inside one 16-B chunk: swizzle the chunk (kv_swz)
      put4(g.k_cache + kv + kv_swz(x.pos, x.i), ko0[0], ko0[1], ko0[2], ko0[3]);
      put4(g.k_cache + kv + kv_swz(x.pos, x.i + half), ko1[0], ko1[1], ko1[2], ko1[3]);
      put4(g.v_cache + kv + kv_swz(x.pos, x.i), v0.x, v0.y, v0.z, v0.w);
      put4(g.v_cache + kv + kv_swz(x.pos, x.i + half), v1.x, v1.y, v1.z, v1.w);
    }
  }
  stamp(st, 3);
}

// ------------------------------------------------------------------ accept
// One warp per request: leading run of drafts equal to the target argmax
// (model.cpp:110-134 semantics on real tokens), bonus = target token at the
// first mismatch (slot_engine.cpp:140), commit and KV rollback by length
// (slot_engine.cpp:151-156; model.hpp:26-28).
__global__ void accept_kernel(FwdMeta m, int n_req, int W, const int32_t* list, const int32_t* ssm_of_req,
                              const float* amax_val, const int32_t* amax_idx, int tiles, int T, SlotState st,
                              int32_t* out_acc, int32_t* out_bonus, int32_t* out_comm, int32_t* out_drafts,
                              int32_t* out_target, unsigned long long* emitted) {
  ptx::grid_dep_wait();
  const int r = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (r >= n_req) return;
  const int slot = list[r];
  const int c = st.committed[slot];
  const int q0 = m.req_qstart[r];
  const int32_t* dr = st.drafts + static_cast<size_t>(slot) * W;
  int32_t* hist = st.tokens + static_cast<size_t>(slot) * st.ctx;
  int a = 0;
  bool alive = true;
  int bonus = -1;
  for (int k = 0; k <= W; ++k) {
    int y = row_argmax_warp(amax_val, amax_idx, tiles, T, q0 + k);
    if (y < 0 || y >= tiles * 128) {  // all-NaN target logits: report (status 4)
      if (lane == 0 && m.err && atomicCAS(m.err, 0, 4) == 0) {
        m.err[1] = slot, m.err[2] = -1, m.err[3] = k, m.err[4] = q0 + k;
        __threadfence_system();
      }
      y = 0;
    }
    if (out_target != nullptr && lane == 0) out_target[static_cast<size_t>(r) * (W + 1) + k] = y;
    if (alive) {
      if (k < W && dr[k] == y) {
        ++a;
      } else {
        alive = false;
        bonus = y;
      }
    }
  }
  if (c + W + 1 > st.ctx) {  // the host refuses such rounds; never commit past the slot's context
    if (lane == 0 && m.err) *reinterpret_cast<volatile int32_t*>(m.err) = 2;
    return;
  }
  if (lane == 0) {
    for (int k = 0; k < a; ++k) hist[c + k] = dr[k];
    hist[c + a] = bonus;
    st.committed[slot] = c + a + 1;
    const int j = ssm_of_req[r];
    if (j >= 0) {
      int32_t* len = st.ssm_len + static_cast<size_t>(j) * st.slots + slot;
      if (*len > c + a) *len = c + a;
    }
    if (out_acc) out_acc[r] = a;
    if (out_bonus) out_bonus[r] = bonus;
    if (out_comm) out_comm[r] = c + a + 1;
    if (out_drafts)
      for (int k = 0; k < W; ++k) out_drafts[static_cast<size_t>(r) * W + k] = dr[k];
    if (emitted) atomicAdd(emitted, static_cast<unsigned long long>(a + 1));
  }
}

// ------------------------------------------------------------------ weights
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// Synthetic weights, written in physical order.
//   tiled = 1: GEMM weight layout -- [ceil(rows/128)][ceil(cols/64)] atoms of 128 x 64 bf16,
//              each a contiguous 16-KiB block holding the 128-B-swizzled shared-memory image
//              (16-B chunk c of row r at c ^ (r % 8)); padding rows / columns are zero;
//   tiled = 0: row-major (the embedding, gathered by token).
// Values depend only on the logical (row, col): the oracle restates them row-major.
// emb != nullptr (lm_head): row v also carries g * E[pi^-1(v)] when v's domain (v / dsize)
// is planted (bit set in `mask`); pi maps each domain of dsize ids onto itself
// (oracle/llama_oracle.c planted_params).
__global__ void init_weights_kernel(bf16* w, int64_t rows, int64_t cols, uint64_t stream, float scale,
                                    const bf16* emb, float g, int64_t dsize, int64_t a_inv, int64_t cc, uint32_t mask,
                                    int tiled) {
  const int64_t katoms = (cols + 63) / 64;
  const int64_t prow = tiled ? (rows + 127) / 128 * 128 : rows, pcols = tiled ? katoms * 64 : cols;
  const int64_t total = prow * pcols;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t row, col;
    if (tiled) {
      const int64_t atom = e >> 13, within = e & 8191;
      const int64_t r = within >> 6, pc = within & 63;
      row = (atom / katoms) * 128 + r;
      col = (atom % katoms) * 64 + ((((pc >> 3) ^ (r & 7)) << 3) | (pc & 7));
    } else {
      row = e / cols, col = e % cols;
    }
    if (row >= rows || col >= cols) {
      w[e] = __float2bfloat16_rn(0.f);
      continue;
    }
    const int64_t le = row * cols + col;  // logical element index
    const float u = static_cast<float>(splitmix64(stream + static_cast<uint64_t>(le)) >> 40);
    const float r = __fsub_rn(__fmul_rn(u, 0x1.0p-23f), 1.0f);
    const float a = __fmul_rn(r, scale);
    const int64_t dom = row / dsize, base = dom * dsize;
    if (emb == nullptr || dom >= 32 || !((mask >> dom) & 1u)) {
      w[e] = __float2bfloat16_rn(a);
    } else {
      const int64_t src = base + (a_inv * (((row - base - cc) % dsize) + dsize)) % dsize;
      const float b = __fmul_rn(g, __bfloat162float(emb[src * cols + col]));
      w[e] = __float2bfloat16_rn(__fadd_rn(a, b));
    }
  }
}

// Row-major [rows][cols] bf16 -> tiled GEMM weight layout (kernel tests, external weights).
__global__ void tile_weights_kernel(const bf16* __restrict__ src, bf16* __restrict__ dst, int64_t rows, int64_t cols) {
  const int64_t katoms = (cols + 63) / 64;
  const int64_t total = (rows + 127) / 128 * 128 * katoms * 64;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t atom = e >> 13, within = e & 8191;
    const int64_t r = within >> 6, pc = within & 63;
    const int64_t p = (atom / katoms) * 128 + r;
    const int64_t col = (atom % katoms) * 64 + ((((pc >> 3) ^ (r & 7)) << 3) | (pc & 7));
    dst[e] = (p < rows && col < cols) ? src[p * cols + col] : __float2bfloat16_rn(0.f);
  }
}

// ------------------------------------------------------------------ toy attention (fp64)
// Block per pack row: for each segment and query, the segment's own max and
// exp-sum (split-KV partial); the combine merges them under the request's
// shared max, which is the aggregation of attention.cpp:128-157.
__global__ void toy_attn_kernel(const double* q, const double* k, const double* v, const int32_t* q_off,
                                const int32_t* kv_off, const int32_t* q_rows, const int32_t* seg,
                                const int32_t* row_ptr, const int32_t* row_seg, int dim, int qmax, double* pm,
                                double* pl, double* po) {
  extern __shared__ double sh[];
  double* red = sh;  // [blockDim]
  const int row = blockIdx.x;
  for (int si = row_ptr[row]; si < row_ptr[row + 1]; ++si) {
    const int s = row_seg[si];
    const int rq = seg[5 * s], len = seg[5 * s + 3] - seg[5 * s + 2], off = seg[5 * s + 4];
    const double* kk = k + (static_cast<size_t>(kv_off[rq]) + off) * dim;
    const double* vv = v + (static_cast<size_t>(kv_off[rq]) + off) * dim;
    for (int j = 0; j < q_rows[rq]; ++j) {
      const double* qq = q + (static_cast<size_t>(q_off[rq]) + j) * dim;
      double mx = -INFINITY;
      for (int key = threadIdx.x; key < len; key += blockDim.x) {
        double d = 0.0;
        for (int c = 0; c < dim; ++c) d += qq[c] * kk[static_cast<size_t>(key) * dim + c];
        mx = fmax(mx, d);
      }
      red[threadIdx.x] = mx;
      __syncthreads();
      for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
        __syncthreads();
      }
      mx = red[0];
      __syncthreads();
      // each thread owns output columns; sums over keys are sequential (fixed order)
      const size_t base = (static_cast<size_t>(s) * qmax + j);
      double den = 0.0;
      for (int c = threadIdx.x; c < dim; c += blockDim.x) {
        double num = 0.0;
        den = 0.0;
        for (int key = 0; key < len; ++key) {
          double d = 0.0;
          for (int cc = 0; cc < dim; ++cc) d += qq[cc] * kk[static_cast<size_t>(key) * dim + cc];
          const double f = exp(d - mx);
          den += f;
          num += f * vv[static_cast<size_t>(key) * dim + c];
        }
        po[base * dim + c] = num;
      }
      if (threadIdx.x == 0) {
        if (dim <= 0) den = 0.0;
        pm[base] = mx;
      }
      if (threadIdx.x == 0 && dim > 0) pl[base] = den;
      __syncthreads();
    }
  }
}

__global__ void toy_combine_kernel(const int32_t* q_off, const int32_t* q_rows, const int32_t* req_seg0,
                                   const int32_t* req_nseg, int dim, int qmax, const double* pm, const double* pl,
                                   const double* po, double* out) {
  const int rq = blockIdx.x;
  for (int j = 0; j < q_rows[rq]; ++j) {
    double M = -INFINITY;
    for (int s = req_seg0[rq]; s < req_seg0[rq] + req_nseg[rq]; ++s) M = fmax(M, pm[static_cast<size_t>(s) * qmax + j]);
    double L = 0.0;
    for (int s = req_seg0[rq]; s < req_seg0[rq] + req_nseg[rq]; ++s)
      L += pl[static_cast<size_t>(s) * qmax + j] * exp(pm[static_cast<size_t>(s) * qmax + j] - M);
    for (int c = threadIdx.x; c < dim; c += blockDim.x) {
      double num = 0.0;
      for (int s = req_seg0[rq]; s < req_seg0[rq] + req_nseg[rq]; ++s)
        num += po[(static_cast<size_t>(s) * qmax + j) * dim + c] * exp(pm[static_cast<size_t>(s) * qmax + j] - M);
      out[(static_cast<size_t>(q_off[rq]) + j) * dim + c] = num / L;
    }
  }
}

template <typename K, typename... Args>
void launch_pdl(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
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
  cudaLaunchKernelEx(&cfg, kernel, args...);
}

}  // namespace

void launch_meta(const MetaArgs& a, const SlotState& st, const FwdMeta& m, cudaStream_t s) {
  ensure_smem_optin(reinterpret_cast<const void*>(meta_kernel), kMetaSmem);
  launch_pdl(meta_kernel, dim3(1), dim3(kMetaThreads), kMetaSmem, s, a, st, m);
}

void launch_embed_norm(const bf16* emb, const FwdMeta& m, int T, int D, float eps, float* h, bf16* xn,
                       cudaStream_t s) {
  launch_pdl(embed_norm_kernel, dim3(T), dim3(kRowThreads), D * sizeof(float), s, emb,
             static_cast<const int32_t*>(m.row_tok), D, eps, h, xn);
}

int qkv_epilogue_blocks(int T, int D) {
  return std::min((T * (D / 8) + kRowThreads - 1) / kRowThreads, 2 * device_sms());
}

int swiglu_blocks(int T, int F) {
  return std::min((T * (F / 4) + kSwiG * kRowThreads - 1) / (kSwiG * kRowThreads), 2 * device_sms());
}

void launch_qkv_epilogue(const float* part, const PieceMap& pm, const FwdMeta& m, int T, const AttnGeom& g,
                         const float* rcos, const float* rsin, float* q, cudaStream_t s, unsigned long long* st) {
  const int blocks = qkv_epilogue_blocks(T, g.n_heads * g.head_dim);
  launch_pdl(qkv_epilogue_kernel, dim3(blocks), dim3(kRowThreads), 0, s, part, pm, m, T, g, rcos, rsin, q, st);
}

void launch_resid_norm(const float* part, const PieceMap& pm, int T, int D, float eps, float* h, bf16* xn,
                       cudaStream_t s, unsigned long long* st) {
  if (D <= 4 * 4 * kRowThreads)
    launch_pdl(resid_norm_kernel<4, 4>, dim3(T), dim3(kRowThreads), 0, s, part, pm, T, D, eps, h, xn, st);
  else
    launch_pdl(resid_norm_kernel<8, 1>, dim3(T), dim3(kRowThreads), 0, s, part, pm, T, D, eps, h, xn, st);
}

void launch_swiglu(const float* part, const PieceMap& pm, int T, int F, bf16* act, cudaStream_t s,
                   unsigned long long* st) {
  const int blocks = swiglu_blocks(T, F);
  launch_pdl(swiglu_kernel, dim3(blocks), dim3(kRowThreads), 0, s, part, pm, T, F, act, st);
}

void launch_accept(const FwdMeta& m, int n_req, int window, const int32_t* list, const int32_t* ssm_of_req,
                   const float* amax_val, const int32_t* amax_idx, int tiles, int T, const SlotState& st,
                   int32_t* out_accepted, int32_t* out_bonus, int32_t* out_committed, int32_t* out_drafts,
                   int32_t* out_target, unsigned long long* emitted, cudaStream_t s) {
  const int per_block = 4;
  launch_pdl(accept_kernel, dim3((n_req + per_block - 1) / per_block), dim3(32 * per_block), 0, s, m, n_req, window,
             list, ssm_of_req, amax_val, amax_idx, tiles, T, st, out_accepted, out_bonus, out_committed, out_drafts,
             out_target, emitted);
}

__global__ void swizzle_kv_kernel(const bf16* __restrict__ src, bf16* __restrict__ dst, int64_t rows, int hd,
                                  int ctx) {
  const int64_t total = rows * hd;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / hd;
    const int d = static_cast<int>(e % hd);
    dst[r * hd + kv_swz(static_cast<int>(r % ctx), d)] = src[e];
  }
}

void launch_swizzle_kv(const bf16* src, bf16* dst, int64_t rows, int hd, int ctx, cudaStream_t s) {
  swizzle_kv_kernel<<<148 * 8, 256, 0, s>>>(src, dst, rows, hd, ctx);
}

void launch_init_weights(bf16* w, int64_t rows, int64_t cols, uint64_t stream, float scale, const bf16* emb,
                         float planted_g, int64_t dsize, int64_t A_inv, int64_t Cc, uint32_t mask, int tiled,
                         cudaStream_t s) {
  init_weights_kernel<<<148 * 8, 256, 0, s>>>(w, rows, cols, stream, scale, emb, planted_g, dsize, A_inv, Cc, mask,
                                              tiled);
}

void launch_tile_weights(const bf16* src, bf16* dst, int64_t rows, int64_t cols, cudaStream_t s) {
  tile_weights_kernel<<<148 * 8, 256, 0, s>>>(src, dst, rows, cols);
}

void launch_toy_attention(const double* q, const double* k, const double* v, const int32_t* q_off,
                          const int32_t* kv_off, const int32_t* q_rows, const int32_t* seg, int n_seg,
                          const int32_t* row_ptr, const int32_t* row_seg, int n_rows, const int32_t* req_seg0,
                          const int32_t* req_nseg, int n_req, int dim, int qmax, double* part_m, double* part_l,
                          double* part_o, double* out, cudaStream_t s) {
  (void)n_seg;
  const int threads = 128;
  if (n_rows > 0)
    toy_attn_kernel<<<n_rows, threads, threads * sizeof(double), s>>>(q, k, v, q_off, kv_off, q_rows, seg, row_ptr,
                                                                      row_seg, dim, qmax, part_m, part_l, part_o);
  if (n_req > 0)
    toy_combine_kernel<<<n_req, 128, 0, s>>>(q_off, q_rows, req_seg0, req_nseg, dim, qmax, part_m, part_l, part_o,
                                             out);
}

}  // namespace spin
