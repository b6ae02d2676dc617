// Micro-benchmarks of the mx kernel's per-order building blocks on one B200
// (not part of the product): cycles per call on one SM.
#include <cooperative_groups.h>
#include <cstdio>
#include "../paper_1908_09301_b200/csrc/taylor_mx.cu"
using namespace mpt;
using namespace mpt::mx;

__global__ void __launch_bounds__(512, 1) kb(int W, int reps, long long* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t* col = (int64_t*)sm;                 // 16 x 128
  int32_t* rows = (int32_t*)(sm + 16384) + 16;  // 16 rows x 144
  const int rs = 144;
  for (int w = tid; w < 16 * 128; w += 512) col[w] = ((int64_t)(w * 2654435761u) << 20) ^ (w * 977);
  for (int w = tid; w < 16 * rs; w += 512) rows[w - 16] = (w % rs) < W ? (int32_t)((w * 2654435761u) >> 5) - (1 << 26) : 0;
  __syncthreads();
  Geo g;
  g.W = W; g.KW = W + 1; g.T = W - 3; g.Tc = W - 2; g.ncols = W + 3; g.ncp = (g.ncols + 3) / 4 * 4;
  g.ng = (W - 1 + 3 + 7) / 8; g.rs = rs;
  MacCount mc;
  // 1. one warp, one product
  long long t0, t1;
  if (warp == 0) {
    t0 = clock64();
    for (int r = 0; r < reps; r++)
      warp_product<8>(rows, make_int2(0, W - 1), rows + rs, make_int2(0, W), g.Tc, g, col + 8 * 128, nullptr);
    t1 = clock64();
    if (lane == 0) out[0] = (t1 - t0) / reps;
  }
  __syncthreads();
  // 2. 15 warps, one product each
  t0 = clock64();
  for (int r = 0; r < reps; r++) {
    if (warp < 15)
      warp_product<8>(rows + (warp % 3) * rs, make_int2(0, W - 1), rows + (3 + warp % 8) * rs, make_int2(0, W), g.Tc, g,
                      col + (warp % 16) * 128, nullptr);
    __syncthreads();
  }
  t1 = clock64();
  if (tid == 0) out[1] = (t1 - t0) / reps;
  // 3. warp_snf on one warp
  if (warp == 0) {
    int2 inf;
    t0 = clock64();
    bool o = false;
    for (int r = 0; r < reps; r++) o |= warp_snf_call<2>(col, g.ncols, W, rows + 12 * rs, &inf);
    t1 = clock64();
    if (lane == 0) { out[2] = (t1 - t0) / reps; out[7] = o; }
  }
  __syncthreads();
  // 4. mac_block alone: 2 blocks of 8 p-steps
  if (warp == 0) {
    int64_t a1[8];
    for (int r = 0; r < 8; r++) a1[r] = 0;
    t0 = clock64();
    for (int r = 0; r < reps; r++) { mac_block(a1, rows, rows + rs, 60 + (lane & 7), lane & 3, (lane & 3) + 12); mac_block(a1, rows, rows + rs, 60 + (lane & 7), (lane & 3) + 8, (lane & 3) + 12); }
    t1 = clock64();
    long long s = 0;
    for (int r = 0; r < 8; r++) s += a1[r];
    if (lane == 0) { out[3] = (t1 - t0) / reps; out[6] = s; }
  }
  __syncthreads();
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  cudaMemset(d, 0, 64);
  cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int W : {8, 62}) {
    kb<<<1, 512, 200 * 1024>>>(W, 50, d);
    long long h[8];
    cudaError_t e = cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    printf("{\"W\": %d, \"warp_product_1warp\": %lld, \"warp_product_15warps\": %lld, \"warp_snf\": %lld, \"mac_block_x2\": %lld, \"err\": \"%s\"}\n",
           W, h[0], h[1], h[2], h[3], cudaGetErrorString(e));
  }
  return 0;
}
