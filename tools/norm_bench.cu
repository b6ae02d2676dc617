// Latency of one normalisation (cycles, clock64) on an otherwise idle SM:
// warp_normalize (1 warp) and group_normalize (4 warps), column counts of
// the K=500 / 2200 / 4200 configurations.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xptxas -v -o tools/norm_bench tools/norm_bench.cu
#include <cstdio>
#include <cstdint>
#include "../paper_1908_09301_b200/csrc/mpt_device.cuh"
using namespace mpt;
__global__ void kb(int ncols, int drop, int W, int group, long long* cyc, int iters) {
  __shared__ int2 info;
  __shared__ int64_t xs[64];
  __shared__ int64_t scol[1024];
  __shared__ int32_t sout[1024];
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) scol[c] = ((int64_t)(c * 2654435761u) << 20) ^ (c * 977);
  __syncthreads();
  long long best = 1LL << 60, tot = 0;
  for (int it = 0; it < iters; it++) {
    __syncthreads();
    long long t0 = clock64();
    bool o;
    if (group == 2)
      o = warp_snf(scol, ncols, W, sout, &info);
    else if (group == 3)
      o = group_normalize_t<2>(scol, ncols, drop, W, sout, threadIdx.x >> 5, blockDim.x >> 5, 1, xs);
    else if (group)
      o = group_normalize(scol, ncols, drop, W, sout, &info, 0, threadIdx.x >> 5, blockDim.x >> 5, 1, xs);
    else
      o = warp_normalize(scol, ncols, drop, W, sout, &info, 0);
    __syncthreads();
    long long dt = clock64() - t0;
    if (o) sout[0] ^= 1;
    best = dt < best ? dt : best;
    tot += dt;
  }
  if (threadIdx.x == 0) {
    cyc[0] = best;
    cyc[1] = tot / iters;
  }
}
int main(int argc, char** argv) {
  long long* d;
  if (argc > 1) {  // profiling mode: one configuration, many iterations
    cudaMalloc(&d, 16);
    kb<<<1, 32>>>(66, 2, 62, 2, d, 2000);
    cudaDeviceSynchronize();
    return 0;
  }
  cudaMalloc(&d, 16);
  int cases[][2] = {{66, 62}, {130, 126}, {266, 263}, {506, 501}};
  for (auto& c : cases) {
    for (int g = 0; g < 4; g++) {
      if (g == 3 && c[0] > 66) continue;
      kb<<<1, (g == 1 || g == 3) ? 128 : 32>>>(c[0], 2, c[1], g, d, 50);
      long long h[2];
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("ncols %d W %d %s: best %lld avg %lld cycles\n", c[0], c[1], g == 0 ? "warp" : g == 1 ? "group4" : g == 2 ? "warp_snf" : "group_t<2>", h[0], h[1]);
    }
  }
  return 0;
}
