// Single-warp latency of the chain building blocks (cycles, clock64):
// warp_product (truncated digit product into columns) and warp_normalize.
#include <cstdio>
#include <cstdint>
#include "../paper_1908_09301_b200/csrc/mpt_device.cuh"
using namespace mpt;
constexpr int kPch = 3;

__device__ __noinline__ void warp_product(const int32_t* A, int2 ia, const int32_t* B, int2 ib, int T, int gf, int ng,
                                          int ncol, int ncx, uint32_t* wsc, int64_t* wcar, int64_t* out) {
  const int lane = threadIdx.x & 31;
  for (int e = lane; e < ng * kPch; e += 32) {
    const int grp = e / kPch, pc = e - grp * kPch;
    const int c0 = kR * (gf + grp);
    Acc acc;
    acc_zero(acc);
    int2 ja = ia;
    const int plo = max(ia.x, c0 - ib.y), phi = min(ia.y, c0 + kR - 1 - ib.x);
    if (plo <= phi) {
      const int b0 = plo / kR, nb = phi / kR - b0 + 1;
      const int per = (nb + kPch - 1) / kPch;
      const int blo = b0 + pc * per, bhi = min(b0 + nb, blo + per) - 1;
      if (blo <= bhi) {
        ja.x = max(ia.x, blo * kR);
        ja.y = min(ia.y, bhi * kR + kR - 1);
        int cnt = 0;
        mac_group(acc, cnt, A, ja, B, ib, c0, T, nullptr);
        acc_fold(acc, c0, T);
      }
    }
    for (int r = 0; r < kR; r++) {
      const int c = c0 + r - T;
      if (c >= 0) wsc[(size_t)pc * ncx + c] = (uint32_t)acc.v[r];
    }
    wcar[(size_t)pc * (ng + 1) + grp] = acc.v[kR];
  }
  __syncwarp();
  for (int c = lane; c < ncol; c += 32) {
    const int cabs = c + T;
    const int own = cabs / kR - gf;
    const int cgb = (cabs % kR == 0) ? cabs / kR - 1 - gf : -1;
    int64_t s = 0;
    if (own >= 0 && own < ng)
      for (int u = 0; u < kPch; u++) s += wsc[(size_t)u * ncx + c];
    if (cgb >= 0 && cgb < ng)
      for (int u = 0; u < kPch; u++) s += wcar[(size_t)u * (ng + 1) + cgb];
    out[c] = s;
  }
  __syncwarp();
}

__global__ void k(int W, long long* out) {
  __shared__ int32_t A[2048], B[2048];
  __shared__ uint32_t wsc[2048];
  __shared__ int64_t wcar[512], cols[1024];
  __shared__ int32_t res[1024];
  __shared__ int2 info;
  const int lane = threadIdx.x;
  for (int d = lane; d < 2048; d += 32) {
    A[d] = (d >= 16 && d < 16 + W) ? ((d * 2654435761u) >> 5) : 0;
    B[d] = (d >= 16 && d < 16 + W) ? ((d * 40503u) & 0xfffffff) : 0;
  }
  __syncwarp();
  const int Lf = W - 1, T = Lf - 2, gf = T / kR, ng = (2 * Lf) / kR - gf + 1;
  const int ncol = kR * (gf + ng) - T + 1, ncx = kR * (ng + 2);
  long long t0 = clock64();
  for (int it = 0; it < 10; it++)
    warp_product(A + 16, make_int2(0, W - 1), B + 16, make_int2(0, W - 1), T, gf, ng, ncol, ncx, wsc, wcar, cols);
  long long t1 = clock64();
  for (int it = 0; it < 10; it++) warp_normalize(cols, ncol, 2, W, res, &info, 0);
  long long t2 = clock64();
  if (lane == 0) {
    out[0] = (t1 - t0) / 10;
    out[1] = (t2 - t1) / 10;
  }
}
int main() {
  long long* d;
  cudaMalloc(&d, 16);
  for (int W : {7, 62, 98, 200, 264, 501}) {
    k<<<1, 32>>>(W, d);
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("W=%d  warp_product %lld cycles   warp_normalize %lld cycles\n", W, h[0], h[1]);
  }
  return 0;
}
