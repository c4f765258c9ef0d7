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
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
