// Micro-benchmark of the mx lead's product stage on one SM (not part of the
// product): 15 warps x one W-digit truncated product each, as in one order.
#include <cstdio>
#include "../paper_1908_09301_b200/csrc/taylor_mx.cu"
using namespace mpt;
using namespace mpt::mx;

template <int NCH>
__global__ void __launch_bounds__(512, 1) kb(int W, int reps, long long* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ Prod slot[16][4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t* col = (int64_t*)sm;                  // 16 x 128
  int32_t* rows = (int32_t*)(sm + 16384) + 16;  // 16 rows x 144
  const int rs = 144;
  for (int w = tid; w < 16 * 128; w += 512) col[w] = 0;
  for (int w = tid; w < 16 * rs; w += 512) rows[w - 16] = (w % rs) < W ? (int32_t)((w * 2654435761u) >> 5) - (1 << 26) : 0;
  __syncthreads();
  Geo g;
  g.W = W; g.KW = W + 1; g.T = W - 3; g.Tc = W - 2; g.ncols = W + 3; g.ncp = (g.ncols + 3) / 4 * 4;
  g.ng = (W - 1 + 3 + 7) / 8; g.rs = rs;
  long long t0 = clock64();
  for (int r = 0; r < reps; r++) {
    if (warp < 15)
      warp_product<NCH>(slot[warp], rows + (warp % 3) * rs, make_int2(0, W - 1), rows + (3 + warp % 8) * rs,
                        make_int2(0, W), g.Tc, g, col + (warp % 16) * 128, nullptr);
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / reps;
  t0 = clock64();
  for (int r = 0; r < reps; r++) {
    if (warp == 0)
      warp_product<NCH>(slot[warp], rows, make_int2(0, W - 1), rows + 3 * rs, make_int2(0, W), g.Tc, g, col, nullptr);
    __syncthreads();
  }
  t1 = clock64();
  if (tid == 0) out[1] = (t1 - t0) / reps;
  if (warp == 0) {
    int2 inf;
    t0 = clock64();
    bool o = false;
    for (int r = 0; r < reps; r++) o |= warp_snf_call<2>(col, g.ncols, W, rows + 12 * rs, &inf);
    t1 = clock64();
    if (lane == 0) { out[2] = (t1 - t0) / reps; out[7] = o; }
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  for (int W : {8, 62}) {
    cudaMemset(d, 0, 64);
    if (W == 8) {
      cudaFuncSetAttribute(kb<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      kb<16><<<1, 512, 200 * 1024>>>(W, 50, d);
    } else {
      cudaFuncSetAttribute(kb<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      kb<8><<<1, 512, 200 * 1024>>>(W, 50, d);
    }
    long long h[8];
    cudaError_t e = cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    printf("{\"W\": %d, \"products_15warps\": %lld, \"product_1warp\": %lld, \"warp_snf\": %lld, \"err\": \"%s\"}\n", W,
           h[0], h[1], h[2], cudaGetErrorString(e));
  }
  return 0;
}
