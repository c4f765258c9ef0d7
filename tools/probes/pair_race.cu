// Does the CTA-pair (cta_group::2) projection GEMM stay correct while other tcgen05 GEMMs
// (cta_group::1, e.g. the SSM draft lm_head with a small ring, two CTAs per SM) run
// concurrently on another stream? Stream A repeats a pair GEMM (PARTIAL) and compares its
// partial buffer bit for bit with the first (quiet) run; stream B keeps argmax GEMMs in flight.
//
// nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a -I../../include -I../../paper_2503_15921_b200/csrc \
//   pair_race.cu -o bin/pair_race -L../../paper_2503_15921_b200 -lspin -Xlinker -rpath,'$ORIGIN/../../../paper_2503_15921_b200'
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "gemm.cuh"
#include "kernels.cuh"

using namespace spin;

__global__ void cmp_kernel(const float* a, const float* b, size_t n, unsigned long long* bad) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned x = __float_as_uint(a[i]), y = __float_as_uint(b[i]);
    if (x != y) atomicAdd(bad, 1ull);
  }
}

int main(int argc, char** argv) {
  const int n_out = argc > 1 ? atoi(argv[1]) : 2304, k = argc > 2 ? atoi(argv[2]) : 768;
  const int t = argc > 3 ? atoi(argv[3]) : 400, iters = argc > 4 ? atoi(argv[4]) : 200;
  const int noise = argc > 5 ? atoi(argv[5]) : 1;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  GemmPlan p = gemm_plan(n_out, k, t, kGemmPartial, sms);
  printf("pair plan: pair %d ntg %d grid %d bn %d max_pieces %d stages %d\n", p.map.pair, p.map.ntg, p.grid, p.bn,
         p.max_pieces, p.stages);
  bf16 *w, *x;
  float *part, *ref;
  cudaMalloc(&w, tiled_weight_elems(n_out, k) * 2);
  cudaMalloc(&x, (size_t)t * k * 2);
  const size_t np = (size_t)p.max_pieces * t * n_out;
  cudaMalloc(&part, np * 4);
  cudaMalloc(&ref, np * 4);
  launch_init_weights(w, n_out, k, 0x1234, 0.05f, nullptr, 0.f, 1, 0, 0, 0u, 1, 0);
  launch_init_weights(x, t, k, 0x99, 1.f, nullptr, 0.f, 1, 0, 0, 0u, 0, 0);
  // the piece table is not needed by the GEMM itself
  GemmEpilogue e;
  e.mode = kGemmPartial;
  e.part = part;
  cudaStream_t sa, sb;
  cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking);
  cudaMemsetAsync(part, 0xff, np * 4, sa);  // NaN fill: slots the GEMM never writes stay NaN in both
  if (gemm_launch(p, w, x, e, sa, true) != cudaSuccess) { printf("launch failed\n"); return 1; }
  cudaMemcpyAsync(ref, part, np * 4, cudaMemcpyDeviceToDevice, sa);
  cudaStreamSynchronize(sa);
  printf("quiet run: %s\n", cudaGetErrorString(cudaGetLastError()));
  // noise: argmax GEMMs like the SSM draft lm_head (V x 768, 16..32 rows, small ring)
  const int nv = 32000, tv = 16;
  GemmPlan ph = gemm_plan(nv, k, tv, kGemmArgmax, sms);
  bf16 *wh, *xh;
  float* av;
  int* ai;
  cudaMalloc(&wh, tiled_weight_elems(nv, k) * 2);
  cudaMalloc(&xh, (size_t)tv * k * 2);
  cudaMalloc(&av, (size_t)ph.n_mtiles * tv * 4);
  cudaMalloc(&ai, (size_t)ph.n_mtiles * tv * 4);
  launch_init_weights(wh, nv, k, 0x77, 0.05f, nullptr, 0.f, 1, 0, 0, 0u, 1, sb);
  launch_init_weights(xh, tv, k, 0x78, 1.f, nullptr, 0.f, 1, 0, 0, 0u, 0, sb);
  GemmEpilogue eh;
  eh.mode = kGemmArgmax;
  eh.amax_val = av;
  eh.amax_idx = ai;
  unsigned long long* bad;
  cudaMallocManaged(&bad, 8);
  *bad = 0;
  cudaDeviceSynchronize();
  for (int i = 0; i < iters; ++i) {
    if (noise)
      for (int r = 0; r < 4; ++r) gemm_launch(ph, wh, xh, eh, sb, true);
    cudaMemsetAsync(part, 0xff, np * 4, sa);
    gemm_launch(p, w, x, e, sa, true);
    cmp_kernel<<<148, 256, 0, sa>>>(part, ref, np, bad);
  }
  cudaDeviceSynchronize();
  printf("iters %d noise %d: mismatching partial words %llu (%s)\n", iters, noise, *bad,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
