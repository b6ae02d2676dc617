// Micro-benchmark of the mx lead's product stage on one SM (not part of the
// product): 15 W-digit truncated products, as in one order, with the one-
// product-per-warp routine (warp_prods) and the several-products-per-warp
// routine (warp_multi).
#include <cstdio>
#include "../paper_1908_09301_b200/csrc/taylor_mx.cu"
using namespace mpt;
using namespace mpt::mx;

template <int NCH, int NP2>
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
  // several products per warp
  const int ppw = 32 / (2 * NP2);
  const int nw = (15 + ppw - 1) / ppw;
  if (warp < nw && lane < ppw) {
    const int pi = warp * ppw + lane;
    if (pi < 15) slot[warp][lane] = mkprod(rows + (pi % 3) * rs, make_int2(0, W - 1), rows + (3 + pi % 8) * rs, make_int2(0, W));
  }
  __syncthreads();
  t0 = clock64();
  for (int r = 0; r < reps; r++) {
    if (warp < nw) {
      const int np = min(ppw, 15 - warp * ppw);
      warp_multi<NP2>(slot[warp], np, g.Tc, g.ng, smem_u32(col + warp * ppw * 128), 128 * 8, g.ncp, g.ncols, nullptr);
    }
    __syncthreads();
  }
  t1 = clock64();
  if (tid == 0) out[1] = (t1 - t0) / reps;
  out[2] = nw;
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  for (int W : {8, 62}) {
    cudaMemset(d, 0, 64);
    if (W == 8) {
      cudaFuncSetAttribute(kb<16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      kb<16, 1><<<1, 512, 200 * 1024>>>(W, 50, d);
    } else {
      cudaFuncSetAttribute(kb<8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      kb<8, 4><<<1, 512, 200 * 1024>>>(W, 50, d);
    }
    long long h[8];
    cudaError_t e = cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    printf("{\"W\": %d, \"one_product_per_warp_15\": %lld, \"multi_products_15\": %lld, \"multi_warps\": %lld, \"err\": \"%s\"}\n",
           W, h[0], h[1], h[2], cudaGetErrorString(e));
  }
  return 0;
}
