// Read-stream ceiling probe: every CTA streams a contiguous slice of a large buffer
// into a shared-memory ring with TMA (1-D bulk copies or 2-D tensor boxes), one
// elected thread issuing, mbarrier completion, nothing computed. Reports GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sp stream_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c));
}
__device__ __forceinline__ void expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(sa(b)),
               "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
               "l"(src), "r"(bytes), "r"(sa(b)) : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* b, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(sa(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(sa(b)) : "memory");
}

// mode 0: 1-D bulk copies of `chunk` bytes; mode 1: 2-D boxes 64 cols x rows (row stride 8 KB, like W tiles)
__global__ void stream(const uint8_t* buf, size_t per_cta, int chunk, int stages, int mode,
                       const __grid_constant__ CUtensorMap tm, int rows_per_box) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + stages * chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t base = blockIdx.x * per_cta;
  const int n = static_cast<int>(per_cta / chunk);
  for (int i = 0; i < n + stages; ++i) {
    if (i >= stages) wait(&bars[(i - stages) % stages], ((i - stages) / stages) & 1);
    if (i < n) {
      const int s = i % stages;
      expect(&bars[s], chunk);
      if (mode == 0) {
        bulk(sm + s * chunk, buf + base + static_cast<size_t>(i) * chunk, chunk, &bars[s]);
      } else {
        // chunk = boxes of 128 B x rows_per_box; CTA owns a 128-row band, walks K
        const int boxes = chunk / (128 * rows_per_box);
        for (int bx = 0; bx < boxes; ++bx)
          tma2d(sm + s * chunk + bx * 128 * rows_per_box, &tm, &bars[s], (i * boxes + bx) * 64,
                blockIdx.x * rows_per_box);
      }
    }
  }
}

int main() {
  const size_t total = 4ull << 30;  // 4 GiB
  uint8_t* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a), cudaEventCreate(&b);
  const int grid_opts[] = {148, 296};
  struct Case { int mode, chunk, stages, rows; };
  const Case cases[] = {{0, 16384, 4, 0}, {0, 16384, 8, 0}, {0, 16384, 12, 0}, {0, 32768, 6, 0}, {0, 65536, 3, 0},
                        {0, 4096, 16, 0}, {1, 16384, 4, 128}, {1, 16384, 8, 128}, {1, 16384, 12, 128}, {1, 32768, 6, 128},
                        {1, 65536, 3, 128}};
  for (int grid : grid_opts)
    for (const Case& c : cases) {
      if (grid == 296 && c.stages * c.chunk > 110 * 1024) continue;
      const size_t per_cta = (total / grid) / 65536 * 65536;
      CUtensorMap tm{};
      // 2-D view: rows of 8 KB (like a 4096-wide bf16 weight), grid*128 rows
      const uint64_t cols = 4096, rows = total / (cols * 2);
      cuuint64_t dims[2] = {cols, rows};
      cuuint64_t str[1] = {cols * 2};
      cuuint32_t box[2] = {64, static_cast<cuuint32_t>(c.rows ? c.rows : 128)};
      cuuint32_t es[2] = {1, 1};
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      // mode 1: each CTA reads its 128-row band over K: per_cta bytes = 128 rows x K2 bytes
      size_t pc = per_cta;
      if (c.mode == 1) pc = std::min<size_t>(per_cta, 128ull * 8192);  // a band holds 1 MiB
      const size_t smem = static_cast<size_t>(c.stages) * c.chunk + 64 * 8;
      stream<<<grid, 32, smem>>>(buf, pc, c.chunk, c.stages, c.mode, tm, c.rows);
      cudaEventRecord(a);
      const int reps = c.mode == 1 ? 20 : 1;
      for (int r = 0; r < reps; ++r) stream<<<grid, 32, smem>>>(buf, pc, c.chunk, c.stages, c.mode, tm, c.rows);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = static_cast<double>(pc) * grid * reps;
      printf("grid %3d mode %d chunk %6d stages %2d inflight/CTA %4d KB: %7.0f GB/s  (%s)\n", grid, c.mode, c.chunk,
             c.stages, c.stages * c.chunk / 1024, bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
