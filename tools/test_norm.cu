// Device unit test of warp_normalize and group_normalize (mpt_device.cuh):
// normalise column vectors read from stdin, print overflow flag + digits,
// once with one warp and once with a 4-warp group (two output lines per case).
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../paper_1908_09301_b200/csrc/mpt_device.cuh"
using namespace mpt;
__global__ void kw(const int64_t* col, int ncols, int drop, int W, int32_t* out, int* ovf) {
  __shared__ int2 info;
  bool o = warp_normalize(col, ncols, drop, W, out, &info, 0);
  if (threadIdx.x == 0) *ovf = o;
}
__global__ void kg(const int64_t* col, int ncols, int drop, int W, int32_t* out, int* ovf) {
  __shared__ int2 info;
  __shared__ int64_t xs[64];
  __shared__ int64_t scol[1024];
  __shared__ int32_t sout[1024];
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) scol[c] = col[c];
  __syncthreads();
  bool o = group_normalize(scol, ncols, drop, W, sout, &info, 0, threadIdx.x >> 5, blockDim.x >> 5, 1, xs);
  __syncthreads();
  for (int d = threadIdx.x; d < W; d += blockDim.x) out[d] = sout[d];
  if (threadIdx.x == 0) *ovf = o;
}
int main() {
  int ncols, drop, W;
  while (scanf("%d %d %d", &ncols, &drop, &W) == 3) {
    std::vector<long long> c(ncols);
    for (int i = 0; i < ncols; i++)
      if (scanf("%lld", &c[i]) != 1) return 1;
    int64_t* dc;
    int32_t* dout;
    int* dov;
    cudaMalloc(&dc, 8 * ncols);
    cudaMalloc(&dout, 4 * (W + 64));
    cudaMalloc(&dov, 4);
    cudaMemcpy(dc, c.data(), 8 * ncols, cudaMemcpyHostToDevice);
    for (int v = 0; v < 2; v++) {
      if (v == 0)
        kw<<<1, 32>>>(dc, ncols, drop, W, dout, dov);
      else
        kg<<<1, 128>>>(dc, ncols, drop, W, dout, dov);
      std::vector<int> out(W);
      int ov;
      cudaMemcpy(out.data(), dout, 4 * W, cudaMemcpyDeviceToHost);
      cudaMemcpy(&ov, dov, 4, cudaMemcpyDeviceToHost);
      printf("%d", ov);
      for (int i = 0; i < W; i++) printf(" %d", out[i]);
      printf("\n");
    }
    cudaFree(dc);
    cudaFree(dout);
    cudaFree(dov);
  }
  return 0;
}
