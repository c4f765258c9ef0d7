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

  int rank;            // CTA pairs: this CTA's weight tile within the pair's super tile

  __device__ void init(const PieceMap& pm, int n_tiles) {
    const int id = static_cast<int>(blockIdx.x) / pm.pair;  // both CTAs of a pair: same schedule
    rank = static_cast<int>(blockIdx.x) % pm.pair;
    grp = pm.ntg > 1 ? id / pm.ntg : id;
    my_nt = pm.ntg > 1 ? id % pm.ntg : 0;
    const long long c = grp;
    u = c * pm.units / pm.grid;
    u_end = (c + 1) * pm.units / pm.grid;
    next_tile = blockIdx.x;
    (void)n_tiles;
  }
  __device__ bool next(const PieceMap& pm, int n_tiles, Piece& p) {
    if (pm.mode == kGemmPartial) {
      if (u >= u_end) return false;
      const int t = static_cast<int>(u / pm.kb);  // tile, or weight tile when grouped (super tiles when paired)
      if (pm.pair == 1) {
        p.tile = pm.ntg > 1 ? t * pm.n_ntiles + my_nt : t;
      } else {
        const int smt = pm.ntg > 1 ? t : t / pm.n_ntiles, nt = pm.ntg > 1 ? my_nt : t % pm.n_ntiles;
        p.tile = (smt * pm.pair + rank) * pm.n_ntiles + nt;
      }
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

// P2 = CTA pair (cta_group::2): the two CTAs of a cluster own the weight tiles 2s and 2s + 1
// of a 256-row super tile; the leader issues one tcgen05.mma M = 256 per k step that reads
// A from both CTAs (128 rows each) and the token tile B split across them (bn / 2 tokens
// each), and writes each CTA's 128 x bn accumulator into that CTA's TMEM. Every SM then
// ingests 16 KB of weights + bn * 64 B of tokens per stage instead of 16 KB + bn * 128 B:
// the single-CTA k-loop was bound by the L2 -> SM operand stream at T > 256.
template <bool P2>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __nv_bfloat16* __restrict__ w_tiled, const __grid_constant__ CUtensorMap tm_x,
                   const __grid_constant__ CUtensorMap tm_part, const __grid_constant__ CUtensorMap tm_w, PieceMap pm,
                   GemmEpilogue epi, int n_out, int t_total, int stages) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);

  const int bn = pm.bn;
  // token rows held (and loaded) per CTA and stage: all bn, or this CTA's half in a pair
  const int bn_cta = P2 ? bn / 2 : bn;
  const uint32_t tile_b_bytes = static_cast<uint32_t>(bn_cta) * kBlockK * 2;
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
  const bool leader = !P2 || (blockIdx.x & 1) == 0;  // cluster rank 0 issues the pair's MMAs
  // stamps [CTA][8]: start, producer wait release, first stage ready (MMA), last MMA issued,
  // first epilogue start, last epilogue done, end
  unsigned long long* st = epi.st ? epi.st + 8 * blockIdx.x : nullptr;
  if (st && threadIdx.x == 0) st[0] = ptx::globaltimer();
  const int n_tiles = pm.n_mtiles * ((t_total + bn - 1) / bn);
  uint32_t tmem_cols = 32;
  while (tmem_cols < static_cast<uint32_t>(2 * bn)) tmem_cols <<= 1;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tm_x);
    if (P2) ptx::tma_prefetch_desc(&tm_w);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull_bar[s], 1);
      ptx::mbar_init(&tempty_bar[s], P2 ? 8 : 4);  // pair: both CTAs' epilogue warps drain the leader's MMA
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) {
    if (P2)
      ptx::tmem_alloc_2sm(tmem_slot, tmem_cols);
    else
      ptx::tmem_alloc(tmem_slot, tmem_cols);
  }
  ptx::tc_fence_before();
  if (P2) {  // the peer signals our barriers and its MMAs write our TMEM
    ptx::cluster_arrive();
    ptx::cluster_wait();
  } else {
    __syncthreads();
  }
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      // weights stream through once (evict-first), unless sibling CTAs of a group re-read them
      const uint64_t pol_w = pm.ntg > 1 ? ptx::policy_evict_last() : ptx::policy_evict_first();
      const uint64_t pol_x = ptx::policy_evict_last();   // activations are re-read by every CTA
      // every stage completes on the leader's full barrier (pair: both CTAs' loads)
      const uint32_t stage_bytes = (kTileABytes + tile_b_bytes) * (P2 ? 2 : 1);
      auto load_a = [&](int s, int mt, int kb) {
        if (P2)
          ptx::tma_load_2d_2sm(smem_a + static_cast<size_t>(s) * kTileABytes, &tm_w,
                               ptx::mapa(ptx::smem_u32(&full_bar[s]), 0), 0, (mt * pm.kb + kb) * kBlockM, pol_w);
        else
          ptx::bulk_load(smem_a + static_cast<size_t>(s) * kTileABytes,
                         w_tiled + (static_cast<size_t>(mt) * pm.kb + kb) * (kBlockM * kBlockK), kTileABytes,
                         &full_bar[s], pol_w);
      };
      PieceIter it;
      it.init(pm, n_tiles);
      Piece p;
      int stage = 0;
      uint32_t phase = 0;
      int prefetched = 0;  // stages whose W half was issued before the dependency wait
      // Issue the weight halves of the first stages before waiting on the
      // producer kernel (PDL): weights never depend on the previous kernel.
      {
        PieceIter pre = it;
        Piece q;
        int s = 0;
        const int pre_n = min(stages, epi.prewait_stages);
        while (s < pre_n && pre.next(pm, n_tiles, q)) {
          const int mt = q.tile / pm.n_ntiles;
          for (int kb = q.kb0; kb < q.kb1 && s < pre_n; ++kb, ++s) {
            if (leader) ptx::mbar_arrive_expect_tx(&full_bar[s], stage_bytes);
            load_a(s, mt, kb);
          }
        }
        prefetched = s;
        // The next k-blocks of the CTA's weight range go to L2 meanwhile (contiguous per
        // piece in the tiled layout: one bulk prefetch per piece), so the stream after the
        // wait starts from L2 instead of HBM (SPIN_GEMM_L2_PREFETCH: blocks per CTA).
        if (!P2 && epi.l2_prefetch_blocks > 0) {
          int left = epi.l2_prefetch_blocks;
          PieceIter pf = it;
          Piece r;
          int skip = prefetched;
          while (left > 0 && pf.next(pm, n_tiles, r)) {
            const int n = r.kb1 - r.kb0;
            if (skip >= n) {
              skip -= n;
              continue;
            }
            const int k0 = r.kb0 + skip, cnt = min(n - skip, left);
            skip = 0;
            left -= cnt;
            const int mt = r.tile / pm.n_ntiles;
            ptx::bulk_prefetch_l2(w_tiled + (static_cast<size_t>(mt) * pm.kb + k0) * (kBlockM * kBlockK),
                                  static_cast<uint32_t>(cnt) * kTileABytes);
          }
        }
      }
      ptx::grid_dep_wait();
      // Early trigger: the dependent (the reduction / epilogue kernel) launches now and its
      // blocks sit resident at their own dependency wait while this grid streams, so the
      // hop after the GEMM costs no launch latency. After our wait, not before: dependents
      // read data of OUR predecessor's predecessor before their wait (resid_norm's h row).
      if (epi.early_trigger) ptx::grid_dep_launch();
      if (st) st[1] = ptx::globaltimer();
      int issued = 0;
      while (it.next(pm, n_tiles, p)) {
        const int mt = p.tile / pm.n_ntiles;
        const int nt = p.tile % pm.n_ntiles;
        for (int kb = p.kb0; kb < p.kb1; ++kb) {
          if (issued >= prefetched) {
            ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
            if (leader) ptx::mbar_arrive_expect_tx(&full_bar[stage], stage_bytes);
            load_a(stage, mt, kb);
          }
          if (P2)  // this CTA's half of the token tile
            ptx::tma_load_2d_2sm(smem_b + static_cast<size_t>(stage) * tile_b_bytes, &tm_x,
                                 ptx::mapa(ptx::smem_u32(&full_bar[stage]), 0), kb * kBlockK,
                                 nt * bn + it.rank * bn_cta, pol_x);
          else
            ptx::tma_load_2d(smem_b + static_cast<size_t>(stage) * tile_b_bytes, &tm_x, &full_bar[stage],
                             kb * kBlockK, nt * bn, pol_x);
          ++issued;
          if (++stage == stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      {
        // producer tail: every stage released by the MMAs (the leader's, in a pair), so no
        // tcgen05.commit arrival is still in flight towards our barriers when the CTA leaves --
        // a late arrival would land in the shared memory of the next CTA on this SM
        for (int i = 0; i < stages; ++i) {
          ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
          if (++stage == stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (pair: leader only)
    if (leader) {
      const uint32_t idesc = ptx::idesc_bf16(P2 ? 256u : 128u, static_cast<uint32_t>(bn));
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
              const uint32_t accum = (kb > p.kb0 || k > 0) ? 1u : 0u;
              if (P2)
                ptx::umma_bf16_2sm(d_addr, da + 2 * k, db + 2 * k, idesc, accum);
              else
                ptx::umma_bf16(d_addr, da + 2 * k, db + 2 * k, idesc, accum);
            }
            if (P2) {  // the stage spans both CTAs: release it in both; the accumulator is in both
              ptx::umma_commit_2sm(&empty_bar[stage], 0x3);
              if (kb + 1 == p.kb1) ptx::umma_commit_2sm(&tfull_bar[acc], 0x3);
            } else {
              ptx::umma_commit(&empty_bar[stage]);
              if (kb + 1 == p.kb1) ptx::umma_commit(&tfull_bar[acc]);
            }
          }
          __syncwarp();
          if (++stage == stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        ++iter;
      }
      if (P2) {
        // accumulator tail: both CTAs' epilogues have drained every accumulator (their
        // remote arrivals on our tempty barriers have landed) before the pair leaves
        for (int i = 0; i < 2; ++i, ++iter) ptx::mbar_wait(&tempty_bar[iter & 1], ((iter >> 1) & 1) ^ 1);
      }
      if (st && lane == 0) st[3] = ptx::globaltimer();
    }
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
    // accumulator release: our own tempty, or the pair leader's
    auto release_acc = [&](int acc) {
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (P2)
          ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&tempty_bar[acc]), 0));
        else
          ptx::mbar_arrive(&tempty_bar[acc]);
      }
    };
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
      if (epi.mode == kGemmPartial) {
        // Each epilogue warp drains its own 32 TMEM lanes (32 output features) and stores
        // them itself: 32-token groups (both 16-token TMEM loads in flight together) staged
        // in the warp's two halves of its staging quarter, one TMA store per 16 tokens x 32
        // features; a half is rewritten only after the warp's group stored from it two
        // groups earlier has been read. No barrier across the epilogue warps.
        static_assert(kStgSlots == 4, "two groups of two 16-token slots per warp");
        float* stg_base = reinterpret_cast<float*>(smem_red) + ew * (kStgSlots * 16 * 32);
        for (int c0 = 0; c0 < bn; c0 += 32, ++chunk) {
          const bool two = c0 + 16 < bn;
          float* stg = stg_base + (chunk & 1) * (2 * 16 * 32);
          if (chunk >= 2) {
            if (lane == 0) ptx::bulk_wait_read<1>();
            __syncwarp();
          }
          uint32_t r[32];
          ptx::tmem_ld16_nowait(t_addr + c0, r);
          if (two) ptx::tmem_ld16_nowait(t_addr + c0 + 16, r + 16);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j) stg[j * 32 + lane] = __uint_as_float(r[j]);
          if (two) {
#pragma unroll
            for (int j = 16; j < 32; ++j) stg[j * 32 + lane] = __uint_as_float(r[j]);
          }
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const int n0 = mt * kBlockM + ew * 32;
            ptx::tma_store_3d(&tm_part, stg, n0, nt * bn + c0, p.slot);
            if (two) ptx::tma_store_3d(&tm_part, stg + 16 * 32, n0, nt * bn + c0 + 16, p.slot);
            ptx::bulk_commit();
          }
        }
        release_acc(acc);
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
        release_acc(acc);
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
    if (epi.mode == kGemmPartial && lane == 0) ptx::bulk_wait0();  // every warp's own stores
    if (st && ew == 0 && lane == 0) st[5] = ptx::globaltimer();
  }

  ptx::grid_dep_launch();
  ptx::tc_fence_before();
  if (P2) {  // neither CTA frees its TMEM / shared memory while the peer may still touch it
    ptx::cluster_arrive();
    ptx::cluster_wait();
  } else {
    __syncthreads();
  }
  ptx::tc_fence_after();
  if (warp == 2) {
    if (P2)
      ptx::tmem_dealloc_2sm(tmem_base, tmem_cols);
    else
      ptx::tmem_dealloc(tmem_base, tmem_cols);
  }
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
  // CTA pairs (cta_group::2, PieceMap::pair) from this many token rows (0 = never): above one
  // token tile (tools/gemm_time_probe.py: T = 1280 QKV 105.3 -> 100.4 us, gate_up 184.9 ->
  // 175.4); at T = 160 the weight stream bounds the k-loop and a pair's coarser stream-K units
  // cost more than the halved token operand saves (QKV 23.2 -> 24.6 us). (A config-4 failure
  // first blamed on pairs was the prewarm race of DESIGN.md section 8: it reproduces with pairs
  // off and not with pairs on once the catch-up waits for the drafts.)
  static const int pair_min_t = [] {
    const char* e = std::getenv("SPIN_GEMM_PAIR_MIN_T");
    return e ? std::atoi(e) : 257;
  }();
  const bool paired = mode == kGemmPartial && pair_min_t > 0 && t >= pair_min_t && p.n_mtiles % 2 == 0 &&
                      p.bn % 32 == 0;
  const size_t stage_bytes = kTileABytes + static_cast<size_t>(paired ? p.bn / 2 : p.bn) * kBlockK * 2;
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
  if (paired) {
    m.pair = 2;
    m.units /= 2;
    num_sms /= 2;  // the stream-K search below runs over CTA pairs
  }
  if (mode == kGemmPartial && p.n_ntiles > 1 && grouped_ok && p.n_ntiles <= num_sms) {
    m.ntg = p.n_ntiles;
    m.units = static_cast<long long>(p.n_mtiles / m.pair) * p.kb;
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
    // The slack counts SMs: with CTA groups of ntg token tiles, one group fewer already idles
    // ntg SMs (T = 1280: 24 instead of 29 groups of 5 left 25 SMs idle for 1 piece per tile,
    // 113 -> 105.6 us for the 7B QKV at 29 groups, tools/gemm_time_probe.py).
    const int gslack = slack / m.ntg;
    if (m.grid == num_sms && m.units <= (1 << 20)) {
      int best = m.grid, best_w = worst(m.grid);
      for (int g = m.grid - 1; g >= m.grid - gslack && g > 0; --g) {
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
  p.grid = m.grid * m.ntg * m.pair;
  return p;
}

cudaError_t gemm_launch(const GemmPlan& plan, const void* W, const void* X, const GemmEpilogue& epi,
                        cudaStream_t stream, bool pdl) {
  CUtensorMap tm_x, tm_part{};
  // paired CTAs each load half of the token tile; their weight atoms come through a 2-D
  // view of the tiled layout ([atoms * 128 rows][64], unswizzled: the atoms already are
  // the swizzled shared-memory images) so that the copy can signal the leader's barrier
  CUtensorMap tm_w{};
  if (!encode_tmap_bf16(&tm_x, X, plan.t, plan.k, plan.bn / plan.map.pair, kBlockK, true)) return cudaErrorInvalidValue;
  if (plan.map.pair > 1 &&
      !encode_tmap_bf16(&tm_w, W, static_cast<uint64_t>(plan.n_mtiles) * plan.kb * kBlockM, kBlockK, kBlockM, kBlockK,
                        false))
    return cudaErrorInvalidValue;
  if (epi.mode == kGemmPartial) {
    // part[slot][t][n_out] fp32 as a 3-D tensor (clips rows t >= T and features n >= n_out)
    auto fn = get_encode_fn();
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(plan.n_out), static_cast<cuuint64_t>(plan.t),
                          static_cast<cuuint64_t>(plan.max_pieces)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(plan.n_out) * 4, static_cast<cuuint64_t>(plan.n_out) * plan.t * 4};
    cuuint32_t box[3] = {32, 16, 1};  // one epilogue warp's staging slot: 32 features x 16 tokens
    cuuint32_t estr[3] = {1, 1, 1};
    if (fn == nullptr || (plan.n_out * 4) % 16 != 0 ||
        fn(&tm_part, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, epi.part, dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const bool p2 = plan.map.pair > 1;
  ensure_smem_optin(p2 ? reinterpret_cast<const void*>(gemm_tc_kernel<true>)
                       : reinterpret_cast<const void*>(gemm_tc_kernel<false>),
                    227 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(plan.grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = plan.smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na++].val.programmaticStreamSerializationAllowed = pdl_allowed();
  }
  if (plan.map.pair > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = plan.map.pair;
    attr[na].val.clusterDim.y = 1;
    attr[na++].val.clusterDim.z = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  GemmEpilogue e = epi;
  static const int early = [] {
    const char* v = std::getenv("SPIN_GEMM_EARLY_TRIGGER");  // A/B switch
    return v ? std::atoi(v) : 0;
  }();
  e.early_trigger = early;
  static const int l2_pf = [] {
    const char* v = std::getenv("SPIN_GEMM_L2_PREFETCH");  // A/B switch: k-blocks per CTA
    return v ? std::atoi(v) : 0;
  }();
  e.l2_prefetch_blocks = plan.map.mode == kGemmPartial ? l2_pf : 0;
  static const int pre_st = [] {
    const char* v = std::getenv("SPIN_GEMM_PREWAIT_STAGES");  // A/B switch (default: the whole ring)
    return v ? std::atoi(v) : (1 << 30);
  }();
  e.prewait_stages = pre_st;
  return cudaLaunchKernelEx(&cfg, p2 ? gemm_tc_kernel<true> : gemm_tc_kernel<false>,
                            static_cast<const __nv_bfloat16*>(W), tm_x, tm_part, tm_w, plan.map, e, plan.n_out, plan.t,
                            plan.stages);
}

}  // namespace spin
