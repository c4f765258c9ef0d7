// Weight-streaming projection GEMM for the verify / draft forward passes.
//
//   Y[t, n] = sum_k X[t, k] * W[n, k]          X: [T, K] bf16, W: [N_out, K] bf16
//
// The weight matrix is the tcgen05 "A" operand (M = 128 output features per
// tile) and the token batch is the "B" operand (N = token tile, 16..256): at
// verification batch sizes (T = B*(gamma+1) = 160) the product is HBM-bound on
// the weight stream, so tiles are cut along the output features and K is split
// stream-K style across all SMs so that every SM pulls 1/148 of the weights.
//
// Two epilogues:
//   * PARTIAL: each CTA writes an fp32 partial sum for the (tile, k-range) piece
//     it owns to part[slot][t][n]; the consumer kernel (residual+RMSNorm,
//     RoPE+KV-append, SwiGLU) reduces the <= max_pieces slots of a tile in a
//     fixed order, so results are deterministic run to run.
//   * ARGMAX: full-K tiles (lm_head); the epilogue reduces each token column to
//     (max logit, lowest index) over its 128 vocabulary rows.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include <vector>

namespace spin {

enum GemmMode : int { kGemmPartial = 0, kGemmArgmax = 1 };

// Stream-K bookkeeping shared by the GEMM and its consumers.
struct PieceMap {
  long long units;  // n_tiles * kb
  int grid;         // CTAs
  int kb;           // 64-wide k blocks per tile
  int n_mtiles;     // 128-row tiles over N_out
  int n_ntiles;     // token tiles; tile = mt * n_ntiles + nt (token tiles of one weight tile adjacent,
                    // so the CTAs streaming them run concurrently and share each weight atom in L2)
  int bn;           // token tile
  int mode;         // GemmMode
  // Grouped stream-K (PARTIAL, more than one token tile): the stream-K units are the
  // weight tiles' k-blocks alone (units = n_mtiles * kb) and `grid` counts CTA GROUPS of
  // ntg = n_ntiles CTAs; the CTAs of a group stream the same weight range at the same
  // time, each against its own token tile, so every weight atom comes from DRAM once and
  // from L2 for its siblings (instead of once per token tile). ntg = 1: plain stream-K.
  int ntg = 1;
  // CTA pairs (PARTIAL): the two CTAs of a 2-CTA cluster own adjacent weight tiles
  // (2s, 2s + 1) over the same token tile and k-range; each TMA-loads half of the token
  // tile and multicasts it to both, so the L2 serves every token tile once per pair. The
  // stream-K units are then the PAIRS' k-blocks (a unit is a 256-row weight super tile).
  int pair = 1;
  const uint8_t* tbl = nullptr;  // device: pieces per tile (filled by the host at plan time)

  // CTA (group, when ntg > 1) that owns stream-K unit u.
  __host__ __device__ __forceinline__ int cta_of(long long u) const {
    return static_cast<int>((u * grid + grid - 1) / units);
  }
  // Number of partial slots written for (token t, feature n).
  __host__ __device__ __forceinline__ int pieces(int t, int n) const {
    if (mode != kGemmPartial) return 1;
    const long long sm = n / (128 * pair);
    const long long tile = ntg > 1 ? sm : sm * n_ntiles + t / bn;
    return cta_of(tile * kb + kb - 1) - cta_of(tile * kb) + 1;
  }
  __device__ __forceinline__ int tile_pieces(int t, int n) const { return tbl[(n / 128) * n_ntiles + t / bn]; }
};

struct GemmPlan {
  int n_out = 0, k = 0, t = 0;
  std::vector<uint8_t> tile_pieces;  // host copy of PieceMap::tbl
  int bn = 0, n_ntiles = 0, n_mtiles = 0, kb = 0;
  int grid = 0, stages = 0, max_pieces = 1;  // grid: CTAs launched (= map.grid * map.ntg * map.pair)
  size_t smem_bytes = 0;
  PieceMap map{};
};

struct GemmEpilogue {
  int mode = kGemmPartial;
  float* part = nullptr;     // PARTIAL: [max_pieces][t][n_out]
  float* amax_val = nullptr; // ARGMAX: [n_mtiles][t]
  int* amax_idx = nullptr;   // ARGMAX: [n_mtiles][t]
  float* logits = nullptr;   // ARGMAX (optional): [t][n_out]
  unsigned long long* st = nullptr;  // optional timeline stamps [CTA][8] (SPIN_STAMPS)
  int early_trigger = 0;             // PDL trigger right after the dependency wait (set by gemm_launch)
  int l2_prefetch_blocks = 0;
  int prewait_stages = 1 << 30;      // ring stages whose weights are issued before the wait        // weight k-blocks beyond the ring prefetched into L2 before the wait
};

// Weights are stored TILED: [ceil(N/128)][ceil(K/64)] atoms of 128 x 64 bf16, each a
// contiguous 16-KiB block that already is the 128-B-swizzled shared-memory image the
// tensor core reads, streamed with 1-D bulk copies: contiguous 16-KiB copies reach
// ~7 TB/s where 2-D boxes over row-major weights (128 B from each of 128 rows 2K bytes
// apart) cap near 5.4 TB/s (profiles/r01_stream_probe.txt).
inline size_t tiled_weight_elems(int64_t rows, int64_t cols) {
  return static_cast<size_t>((rows + 127) / 128) * ((cols + 63) / 64) * 128 * 64;
}

// Plans a launch for the given shape on `num_sms` SMs.
GemmPlan gemm_plan(int n_out, int k, int t, int mode, int num_sms);

// Launches with W in the tiled layout and X row-major [t][k] (TMA box 64 x bn).
// `pdl` enables programmatic dependent launch.
cudaError_t gemm_launch(const GemmPlan& plan, const void* W, const void* X, const GemmEpilogue& epi,
                        cudaStream_t stream, bool pdl);

// Encodes a 2-D bf16 K-major tensor map with 128-B swizzle (rows x cols, box rows x 64).
bool encode_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                      uint32_t box_cols, bool swizzle128);

// Dynamic shared-memory opt-in of `kernel` on the CURRENT device, set once per
// (kernel, device) and raised when a larger size is requested (thread-safe; the
// attribute is per device context, so a second spin_ctx on another GPU needs its own).
cudaError_t ensure_smem_optin(const void* kernel, size_t bytes);

// Programmatic dependent launch on every kernel launch (1), or off everywhere (SPIN_NO_PDL=1,
// debugging: every kernel then waits for its predecessor's completion before it starts).
int pdl_allowed();
cudaError_t upload_sync(void* dst, const void* src, size_t bytes);  // devattr.cpp
cudaError_t zero_sync(void* dst, size_t bytes);

}  // namespace spin
