// Kernel-hop vs grid-barrier latency on one B200 (decides whether a persistent,
// grid-barrier draft-step kernel can beat the launch-per-phase chain).
//
//   A) chain of N tiny PDL kernels (148 CTAs x 256 threads) captured in a CUDA graph:
//      each waits on its predecessor (griddepcontrol.wait), touches one L2 line per CTA,
//      triggers its dependent. -> us per hop
//   B) one persistent kernel (148 CTAs x 256 threads), N grid barriers (arrival counter +
//      generation word, release/acquire at gpu scope), same L2 touch per phase. -> us per barrier
//   C) as B with 296 CTAs (2 per SM).
//
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o hop_probe hop_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void hop_kernel(float* buf, int i) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  if (threadIdx.x == 0) buf[blockIdx.x * 32] += static_cast<float>(i);
}

__device__ __forceinline__ void grid_barrier(unsigned* count, volatile unsigned* gen, unsigned nblocks, unsigned& g) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned want = g + 1;
    unsigned prev;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(count) : "memory");
    if (prev == nblocks * want - 1) {
      asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(gen), "r"(want) : "memory");
    } else {
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(gen) : "memory");
      } while (v < want);
    }
    g = want;
  }
  __syncthreads();
}

__global__ void persistent_kernel(float* buf, unsigned* count, unsigned* gen, int n) {
  unsigned g = 0;
  for (int i = 0; i < n; ++i) {
    if (threadIdx.x == 0) buf[blockIdx.x * 32] += static_cast<float>(i);
    grid_barrier(count, gen, gridDim.x, g);
  }
}

// D/E) realistic phase: every CTA reads the whole 48-KB activation buffer (bf16 32 x 768) written
// by all CTAs in the previous phase, reduces it, writes its slice of the next buffer.
__device__ __forceinline__ void phase_work(const uint4* __restrict__ in, uint4* __restrict__ out, int n16) {
  __shared__ float red[8];
  uint32_t acc = 0;
  for (int i = threadIdx.x; i < n16; i += blockDim.x) {
    uint4 v = __ldcg(in + i);
    acc ^= v.x + v.y + v.z + v.w;
  }
  for (int o = 16; o; o >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = __uint_as_float(acc);
  __syncthreads();
  const int per = (n16 + gridDim.x - 1) / gridDim.x;
  for (int i = threadIdx.x; i < per; i += blockDim.x) {
    const int e = blockIdx.x * per + i;
    if (e < n16) out[e] = make_uint4(__float_as_uint(red[i % 8]) + e, 1, 2, 3);
  }
}

__global__ void work_hop_kernel(uint4* a, uint4* b, int n16) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  phase_work(a, b, n16);
}

__global__ void work_persistent_kernel(uint4* a, uint4* b, unsigned* count, unsigned* gen, int n, int n16) {
  unsigned g = 0;
  for (int i = 0; i < n; ++i) {
    phase_work(i & 1 ? b : a, i & 1 ? a : b, n16);
    grid_barrier(count, gen, gridDim.x, g);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* buf;
  unsigned *count, *gen;
  cudaMalloc(&buf, 4096 * 32 * 4);
  cudaMalloc(&count, 4);
  cudaMalloc(&gen, 4);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int N = 400;

  // A) PDL chain in a graph
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < N; ++i) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, hop_kernel, buf, i);
  }
  cudaStreamEndCapture(s, &graph);
  cudaGraphInstantiate(&exec, graph, 0);
  for (int w = 0; w < 3; ++w) cudaGraphLaunch(exec, s);
  cudaEventRecord(a, s);
  for (int r = 0; r < 10; ++r) cudaGraphLaunch(exec, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("A pdl-graph hop: %.3f us per kernel (%d CTAs)\n", ms * 1000.f / (10 * N), sms);

  // B/C) persistent kernel with grid barriers
  for (int mult = 1; mult <= 2; ++mult) {
    const int grid = sms * mult;
    for (int w = 0; w < 2; ++w) {
      cudaMemsetAsync(count, 0, 4, s);
      cudaMemsetAsync(gen, 0, 4, s);
      persistent_kernel<<<grid, 256, 0, s>>>(buf, count, gen, N);
    }
    cudaMemsetAsync(count, 0, 4, s);
    cudaMemsetAsync(gen, 0, 4, s);
    cudaEventRecord(a, s);
    persistent_kernel<<<grid, 256, 0, s>>>(buf, count, gen, N * 10);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("%c grid barrier: %.3f us per barrier (%d CTAs)\n", mult == 1 ? 'B' : 'C', ms * 1000.f / (10 * N), grid);
  }
  // D) realistic PDL chain, E) realistic persistent
  uint4 *wa, *wb;
  const int n16 = 32 * 768 * 2 / 16;
  cudaMalloc(&wa, n16 * 16);
  cudaMalloc(&wb, n16 * 16);
  cudaMemset(wa, 0, n16 * 16);
  cudaMemset(wb, 0, n16 * 16);
  cudaGraph_t g2;
  cudaGraphExec_t e2;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < N; ++i) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, work_hop_kernel, i & 1 ? wb : wa, i & 1 ? wa : wb, n16);
  }
  cudaStreamEndCapture(s, &g2);
  cudaGraphInstantiate(&e2, g2, 0);
  for (int w = 0; w < 3; ++w) cudaGraphLaunch(e2, s);
  cudaEventRecord(a, s);
  for (int r = 0; r < 10; ++r) cudaGraphLaunch(e2, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("D pdl-graph hop with 48-KB phase work: %.3f us per kernel\n", ms * 1000.f / (10 * N));
  for (int w = 0; w < 2; ++w) {
    cudaMemsetAsync(count, 0, 4, s);
    cudaMemsetAsync(gen, 0, 4, s);
    work_persistent_kernel<<<sms, 256, 0, s>>>(wa, wb, count, gen, N, n16);
  }
  cudaMemsetAsync(count, 0, 4, s);
  cudaMemsetAsync(gen, 0, 4, s);
  cudaEventRecord(a, s);
  work_persistent_kernel<<<sms, 256, 0, s>>>(wa, wb, count, gen, N * 10, n16);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("E persistent with 48-KB phase work: %.3f us per phase\n", ms * 1000.f / (10 * N));
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
