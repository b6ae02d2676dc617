// Device unit test of warp_normalize (mpt_device.cuh): normalise column
// vectors read from stdin, print the digits (used to debug the kernels).
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../paper_1908_09301_b200/csrc/mpt_device.cuh"
using namespace mpt;
__global__ void k(const int64_t* col, int ncols, int drop, int W, int32_t* out, int* ovf) {
  __shared__ int2 info;
  bool o = warp_normalize(col, ncols, drop, W, out, &info, 0);
  if (threadIdx.x == 0) *ovf = o;
}
int main() {
  int ncols, drop, W;
  while (scanf("%d %d %d", &ncols, &drop, &W) == 3) {
    std::vector<long long> c(ncols);
    for (int i = 0; i < ncols; i++) scanf("%lld", &c[i]);
    int64_t* dc; int32_t* dout; int* dov;
    cudaMalloc(&dc, 8 * ncols); cudaMalloc(&dout, 4 * (W + 64)); cudaMalloc(&dov, 4);
    cudaMemcpy(dc, c.data(), 8 * ncols, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(dc, ncols, drop, W, dout, dov);
    std::vector<int> out(W); int ov;
    cudaMemcpy(out.data(), dout, 4 * W, cudaMemcpyDeviceToHost);
    cudaMemcpy(&ov, dov, 4, cudaMemcpyDeviceToHost);
    printf("%d", ov);
    for (int i = 0; i < W; i++) printf(" %d", out[i]);
    printf("\n");
    cudaFree(dc); cudaFree(dout); cudaFree(dov);
  }
  return 0;
}
