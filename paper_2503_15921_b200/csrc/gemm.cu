// tcgen05 / TMEM / TMA weight-streaming GEMM (see gemm.cuh for the contract).
//
// CTA = 8 warps, one CTA per SM (persistent):
//   warp 0      TMA producer (one elected lane): W tile 128x64 (1-D bulk copy of a
//               pre-tiled 16-KiB atom) + X tile bn x64 (2-D tensor map) per stage
//   warp 1      MMA issuer (lane 0): 4 x tcgen05.mma 128 x bn x 16 per stage
//   warp 2      TMEM allocator (2 accumulator buffers of bn fp32 columns)
//   warps 4..7  epilogue: tcgen05.ld 32 lanes each -> partial store / argmax
#include "gemm.cuh"
#include "ptx.cuh"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <mutex>

namespace spin {

namespace {

constexpr int kBlockM = 128;
constexpr int kBlockK = 64;
constexpr int kMaxStages = 8;
constexpr int kThreads = 256;
constexpr uint32_t kTileABytes = kBlockM * kBlockK * 2;  // 16 KiB
constexpr size_t kRedBytes = 4 * 256 * 8;                // argmax cross-warp scratch
// PARTIAL epilogue: fp32 tiles leave through kStgSlots staging slots of 16 tokens x 128
// features (8 KB), one TMA tensor store per slot, so storing a piece neither waits for the
// ring to drain nor competes with the weight stream for LSU bandwidth.
constexpr int kStgSlots = 4;
constexpr size_t kStgBytes = static_cast<size_t>(kStgSlots) * 16 * kBlockM * 4;
constexpr size_t kBarBytes = 256;

struct Piece {
  int tile, kb0, kb1, slot;
};

// Deterministic per-CTA work sequence, identical in every role.
struct PieceIter {
  long long u, u_end;  // stream-K unit range (PARTIAL)
  int next_tile;       // round-robin tile (ARGMAX)
  int grp, my_nt;      // grouped stream-K: this CTA's group and token tile

  __device__ void init(const PieceMap& pm, int n_tiles) {
    grp = pm.ntg > 1 ? static_cast<int>(blockIdx.x) / pm.ntg : static_cast<int>(blockIdx.x);
    my_nt = pm.ntg > 1 ? static_cast<int>(blockIdx.x) % pm.ntg : 0;
    const long long c = grp;
    u = c * pm.units / pm.grid;
    u_end = (c + 1) * pm.units / pm.grid;
    next_tile = blockIdx.x;
    (void)n_tiles;
  }
  __device__ bool next(const PieceMap& pm, int n_tiles, Piece& p) {
    if (pm.mode == kGemmPartial) {
      if (u >= u_end) return false;
      const int t = static_cast<int>(u / pm.kb);  // tile, or weight tile when grouped
      p.tile = pm.ntg > 1 ? t * pm.n_ntiles + my_nt : t;
      p.kb0 = static_cast<int>(u % pm.kb);
      const long long left = u_end - u;
      p.kb1 = static_cast<int>((p.kb0 + left < pm.kb) ? p.kb0 + left : pm.kb);
      p.slot = grp - pm.cta_of(static_cast<long long>(t) * pm.kb);
      u += p.kb1 - p.kb0;
      return true;
    }
    if (next_tile >= n_tiles) return false;
    p.tile = next_tile;
    p.kb0 = 0;
    p.kb1 = pm.kb;
    p.slot = 0;
    next_tile += pm.grid;
    return true;
  }
};

__device__ __forceinline__ void argmax_merge(float& v, int& i, float ov, int oi) {
  if (ov > v || (ov == v && oi < i)) {
    v = ov;
    i = oi;
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __nv_bfloat16* __restrict__ w_tiled, const __grid_constant__ CUtensorMap tm_x,
                   const __grid_constant__ CUtensorMap tm_part, PieceMap pm, GemmEpilogue epi, int n_out, int t_total,
                   int stages) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);

  const int bn = pm.bn;
  const uint32_t tile_b_bytes = static_cast<uint32_t>(bn) * kBlockK * 2;
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + static_cast<size_t>(stages) * kTileABytes;
  uint8_t* smem_red = smem_b + static_cast<size_t>(stages) * tile_b_bytes;  // ARGMAX scratch | PARTIAL staging
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(smem_red + (pm.mode == kGemmPartial ? kStgBytes : kRedBytes));
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + kMaxStages;
  uint64_t* tfull_bar = bars + 2 * kMaxStages;
  uint64_t* tempty_bar = bars + 2 * kMaxStages + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kMaxStages + 4);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  // stamps [CTA][8]: start, producer wait release, first stage ready (MMA), last MMA issued,
  // first epilogue start, last epilogue done, end
  unsigned long long* st = epi.st ? epi.st + 8 * blockIdx.x : nullptr;
  if (st && threadIdx.x == 0) st[0] = ptx::globaltimer();
  const int n_tiles = pm.n_mtiles * ((t_total + bn - 1) / bn);
  uint32_t tmem_cols = 32;
  while (tmem_cols < static_cast<uint32_t>(2 * bn)) tmem_cols <<= 1;

  if (warp == 0 && lane == 0) ptx::tma_prefetch_desc(&tm_x);
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull_bar[s], 1);
      ptx::mbar_init(&tempty_bar[s], 4);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, tmem_cols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      // weights stream through once (evict-first), unless sibling CTAs of a group re-read them
      const uint64_t pol_w = pm.ntg > 1 ? ptx::policy_evict_last() : ptx::policy_evict_first();
      const uint64_t pol_x = ptx::policy_evict_last();   // activations are re-read by every CTA
      PieceIter it;
      it.init(pm, n_tiles);
      Piece p;
      int stage = 0;
      uint32_t phase = 0;
      bool waited = false;
      int prefetched = 0;  // stages whose W half was issued before the dependency wait
      // Issue the weight halves of the first stages before waiting on the
      // producer kernel (PDL): weights never depend on the previous kernel.
      {
        PieceIter pre = it;
        Piece q;
        int s = 0;
        while (s < stages && pre.next(pm, n_tiles, q)) {
          const int mt = q.tile / pm.n_ntiles;
          for (int kb = q.kb0; kb < q.kb1 && s < stages; ++kb, ++s) {
            ptx::mbar_arrive_expect_tx(&full_bar[s], kTileABytes + tile_b_bytes);
            ptx::bulk_load(smem_a + static_cast<size_t>(s) * kTileABytes,
                           w_tiled + (static_cast<size_t>(mt) * pm.kb + kb) * (kBlockM * kBlockK), kTileABytes,
                           &full_bar[s], pol_w);
          }
        }
        prefetched = s;
      }
      ptx::grid_dep_wait();
      waited = true;
      if (st) st[1] = ptx::globaltimer();
      int issued = 0;
      while (it.next(pm, n_tiles, p)) {
        const int mt = p.tile / pm.n_ntiles;
        const int nt = p.tile % pm.n_ntiles;
        for (int kb = p.kb0; kb < p.kb1; ++kb) {
          if (issued >= prefetched) {
            ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
            ptx::mbar_arrive_expect_tx(&full_bar[stage], kTileABytes + tile_b_bytes);
            ptx::bulk_load(smem_a + static_cast<size_t>(stage) * kTileABytes,
                           w_tiled + (static_cast<size_t>(mt) * pm.kb + kb) * (kBlockM * kBlockK), kTileABytes,
                           &full_bar[stage], pol_w);
          }
          ptx::tma_load_2d(smem_b + static_cast<size_t>(stage) * tile_b_bytes, &tm_x, &full_bar[stage],
                           kb * kBlockK, nt * bn, pol_x);
          ++issued;
          if (++stage == stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      (void)waited;
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = ptx::idesc_bf16_m128(static_cast<uint32_t>(bn));
    PieceIter it;
    it.init(pm, n_tiles);
    Piece p;
    int stage = 0;
    uint32_t phase = 0;
    int iter = 0;
    while (it.next(pm, n_tiles, p)) {
      const int acc = iter & 1;
      ptx::mbar_wait(&tempty_bar[acc], ((iter >> 1) & 1) ^ 1);
      ptx::tc_fence_after();
      const uint32_t d_addr = tmem_base + static_cast<uint32_t>(acc * bn);
      for (int kb = p.kb0; kb < p.kb1; ++kb) {
        ptx::mbar_wait(&full_bar[stage], phase);
        ptx::tc_fence_after();
        if (st && lane == 0 && iter == 0 && kb == p.kb0) st[2] = ptx::globaltimer();
        if (lane == 0) {
          const uint64_t da = ptx::smem_desc_sw128(smem_a + static_cast<size_t>(stage) * kTileABytes);
          const uint64_t db = ptx::smem_desc_sw128(smem_b + static_cast<size_t>(stage) * tile_b_bytes);
#pragma unroll
          for (int k = 0; k < kBlockK / 16; ++k) {
            // +32 bytes per 16-element K step inside the 128-B swizzle atom.
            ptx::umma_bf16(d_addr, da + 2 * k, db + 2 * k, idesc, (kb > p.kb0 || k > 0) ? 1u : 0u);
          }
          ptx::umma_commit(&empty_bar[stage]);
          if (kb + 1 == p.kb1) ptx::umma_commit(&tfull_bar[acc]);
        }
        __syncwarp();
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
      }
      ++iter;
    }
    if (st && lane == 0) st[3] = ptx::globaltimer();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 4;  // TMEM lane quadrant (warp % 4)
    ptx::grid_dep_wait();     // outputs may still be read by the previous kernel
    float* red_v = reinterpret_cast<float*>(smem_red);
    int* red_i = reinterpret_cast<int*>(smem_red + 4 * 256 * 4);
    PieceIter it;
    it.init(pm, n_tiles);
    Piece p;
    int iter = 0, chunk = 0;
    while (it.next(pm, n_tiles, p)) {
      const int acc = iter & 1;
      const int mt = p.tile / pm.n_ntiles;
      const int nt = p.tile % pm.n_ntiles;
      ptx::mbar_wait(&tfull_bar[acc], (iter >> 1) & 1);
      ptx::tc_fence_after();
      if (st && ew == 0 && lane == 0 && iter == 0) st[4] = ptx::globaltimer();
      const int row = ew * 32 + lane;
      const int n = mt * kBlockM + row;
      const bool n_ok = n < n_out;
      const uint32_t t_addr = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + static_cast<uint32_t>(acc * bn);
      PieceIter ahead = it;
      Piece pn;
      const bool last_piece = !ahead.next(pm, n_tiles, pn);
      if (epi.mode == kGemmPartial) {
        // 16-token chunks through the staging slots; a slot is rewritten only after the
        // store issued kStgSlots chunks earlier has finished reading it
        float* stg_base = reinterpret_cast<float*>(smem_red);
        for (int c0 = 0; c0 < bn; c0 += 16, ++chunk) {
          float* stg = stg_base + (chunk % kStgSlots) * (16 * kBlockM);
          if (chunk >= kStgSlots) {
            if (ew == 0 && lane == 0) ptx::bulk_wait_read<kStgSlots - 1>();
            asm volatile("bar.sync 1, 128;" ::: "memory");
          }
          float v[16];
          ptx::tmem_ld16(t_addr + c0, v);
#pragma unroll
          for (int j = 0; j < 16; ++j) stg[j * kBlockM + row] = v[j];
          ptx::fence_proxy_async_smem();
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (ew == 0 && lane == 0) {
            ptx::tma_store_3d(&tm_part, stg, mt * kBlockM, nt * bn + c0, p.slot);
            ptx::bulk_commit();
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&tempty_bar[acc]);
        (void)last_piece;
        (void)n_ok;
      } else {
        for (int c0 = 0; c0 < bn; c0 += 16) {
          float v[16];
          ptx::tmem_ld16(t_addr + c0, v);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int t = nt * bn + c0 + j;
            float bv = n_ok ? v[j] : -INFINITY;
            int bi = n_ok ? n : 0x7fffffff;
            if (epi.logits != nullptr && n_ok && t < t_total) epi.logits[static_cast<size_t>(t) * n_out + n] = v[j];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
              const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
              const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
              argmax_merge(bv, bi, ov, oi);
            }
            if (lane == 0) {
              red_v[ew * 256 + c0 + j] = bv;
              red_i[ew * 256 + c0 + j] = bi;
            }
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&tempty_bar[acc]);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        for (int c = ew * 32 + lane; c < bn; c += 128) {
          const int t = nt * bn + c;
          if (t >= t_total) continue;
          float bv = red_v[c];
          int bi = red_i[c];
          for (int w = 1; w < 4; ++w) argmax_merge(bv, bi, red_v[w * 256 + c], red_i[w * 256 + c]);
          epi.amax_val[static_cast<size_t>(mt) * t_total + t] = bv;
          epi.amax_idx[static_cast<size_t>(mt) * t_total + t] = bi;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      if (st && ew == 0 && lane == 0 && iter == 0) st[7] = ptx::globaltimer();
      ++iter;
    }
    // partials must be in global memory before the grid completes (the consumer reads them)
    if (epi.mode == kGemmPartial && ew == 0 && lane == 0) ptx::bulk_wait0();
    if (st && ew == 0 && lane == 0) st[5] = ptx::globaltimer();
  }

  ptx::grid_dep_launch();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc(tmem_base, tmem_cols);
  if (st && threadIdx.x == 0) st[6] = ptx::globaltimer();
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

}  // namespace

bool encode_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                      uint32_t box_cols, bool swizzle128) {
  auto fn = get_encode_fn();
  if (fn == nullptr) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

GemmPlan gemm_plan(int n_out, int k, int t, int mode, int num_sms) {
  GemmPlan p;
  p.n_out = n_out;
  p.k = k;
  p.t = t;
  p.n_ntiles = (t + 255) / 256;
  const int per = (t + p.n_ntiles - 1) / p.n_ntiles;
  p.bn = std::max(16, (per + 15) / 16 * 16);
  p.n_mtiles = (n_out + kBlockM - 1) / kBlockM;
  p.kb = (k + kBlockK - 1) / kBlockK;
  const long long n_tiles = static_cast<long long>(p.n_mtiles) * p.n_ntiles;
  const size_t stage_bytes = kTileABytes + static_cast<size_t>(p.bn) * kBlockK * 2;
  const size_t budget = 227 * 1024 - 1024 - (mode == kGemmPartial ? kStgBytes : kRedBytes) - kBarBytes;
  static const int cap = [] {
    const char* e = std::getenv("SPIN_GEMM_STAGES");  // experiments only
    return e ? std::atoi(e) : kMaxStages;
  }();
  p.stages = static_cast<int>(std::min<size_t>(std::min(kMaxStages, cap), budget / stage_bytes));
  // Draft-step lm_heads (few rows) run beside the other SSM's kernels: a small ring lets
  // CTAs of both co-reside instead of one 227-KB CTA owning each SM.
  static const int small_ring = [] {
    const char* e = std::getenv("SPIN_GEMM_SMALL_RING");  // experiments only
    return e ? std::atoi(e) : 4;
  }();
  if (mode == kGemmArgmax && t <= 32 && small_ring > 0) p.stages = std::min(p.stages, small_ring);
  p.smem_bytes = 1024 + p.stages * stage_bytes + (mode == kGemmPartial ? kStgBytes : kRedBytes) + kBarBytes;
  PieceMap& m = p.map;
  m.mode = mode;
  m.kb = p.kb;
  m.n_mtiles = p.n_mtiles;
  m.n_ntiles = p.n_ntiles;
  m.bn = p.bn;
  m.units = n_tiles * p.kb;
  static const bool grouped_ok = [] {
    const char* e = std::getenv("SPIN_GEMM_GROUPED");  // A/B switch
    return e ? std::atoi(e) != 0 : true;
  }();
  if (mode == kGemmPartial && p.n_ntiles > 1 && grouped_ok && p.n_ntiles <= num_sms) {
    m.ntg = p.n_ntiles;
    m.units = static_cast<long long>(p.n_mtiles) * p.kb;
    num_sms /= m.ntg;  // the stream-K search below runs over CTA groups
  }
  if (mode == kGemmPartial) {
    // At least kMinUnits k-blocks (64 KiB of weights) per CTA: small draft
    // GEMMs then use fewer SMs instead of fragmenting every tile into many
    // partial pieces that the consumer must re-read (4 measured best of 1/2/4/8
    // on the config-2 draft loop).
    constexpr long long kMinUnits = 4;
    m.grid = static_cast<int>(std::min<long long>(num_sms, std::max<long long>(1, (m.units + kMinUnits - 1) / kMinUnits)));
    // A few SMs fewer can cut the worst-case pieces per tile (e.g. 144 CTAs split every
    // 64-k-block QKV tile into exactly 2 pieces where 148 leave some with 3): the consumer
    // re-reads max_pieces partials per element. Search down to grid - kGridSlack.
    static const int slack = [] {
      const char* e = std::getenv("SPIN_GEMM_GRID_SLACK");  // tuning
      return e ? std::atoi(e) : 8;
    }();
    auto worst = [&](int g) {
      PieceMap q = m;
      q.grid = g;
      int w = 1;
      for (long long tile = 0; tile < n_tiles; ++tile)
        w = std::max(w, q.pieces(static_cast<int>((tile % p.n_ntiles) * p.bn), static_cast<int>((tile / p.n_ntiles) * kBlockM)));
      return w;
    };
    if (m.grid == num_sms && m.units <= (1 << 20)) {
      int best = m.grid, best_w = worst(m.grid);
      for (int g = m.grid - 1; g >= m.grid - slack && g > 0; --g) {
        const int w = worst(g);
        if (w < best_w) best = g, best_w = w;
      }
      m.grid = best;
    }
    // Worst-case pieces per tile: a tile spans ceil(kb / per_cta) + 1 CTAs.
    int mp = 1;
    p.tile_pieces.resize(n_tiles);
    for (long long tile = 0; tile < n_tiles; ++tile) {
      const int np = m.pieces(static_cast<int>((tile % p.n_ntiles) * p.bn), static_cast<int>((tile / p.n_ntiles) * kBlockM));
      p.tile_pieces[tile] = static_cast<uint8_t>(np);
      mp = std::max(mp, np);
    }
    p.max_pieces = mp;
  } else {
    m.grid = static_cast<int>(std::min<long long>(num_sms, n_tiles));
    p.max_pieces = 1;
  }
  p.grid = m.grid * m.ntg;
  return p;
}

cudaError_t gemm_launch(const GemmPlan& plan, const void* W, const void* X, const GemmEpilogue& epi,
                        cudaStream_t stream, bool pdl) {
  CUtensorMap tm_x, tm_part{};
  if (!encode_tmap_bf16(&tm_x, X, plan.t, plan.k, plan.bn, kBlockK, true)) return cudaErrorInvalidValue;
  if (epi.mode == kGemmPartial) {
    // part[slot][t][n_out] fp32 as a 3-D tensor (clips rows t >= T and features n >= n_out)
    auto fn = get_encode_fn();
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(plan.n_out), static_cast<cuuint64_t>(plan.t),
                          static_cast<cuuint64_t>(plan.max_pieces)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(plan.n_out) * 4, static_cast<cuuint64_t>(plan.n_out) * plan.t * 4};
    cuuint32_t box[3] = {static_cast<cuuint32_t>(kBlockM), 16, 1};  // one staging slot
    cuuint32_t estr[3] = {1, 1, 1};
    if (fn == nullptr || (plan.n_out * 4) % 16 != 0 ||
        fn(&tm_part, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, epi.part, dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  ensure_smem_optin(reinterpret_cast<const void*>(gemm_tc_kernel), 227 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(plan.grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = plan.smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  GemmEpilogue e = epi;
  return cudaLaunchKernelEx(&cfg, gemm_tc_kernel, static_cast<const __nv_bfloat16*>(W), tm_x, tm_part, plan.map, e,
                            plan.n_out, plan.t, plan.stages);
}

}  // namespace spin
