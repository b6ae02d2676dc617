// Throughput of the Cauchy inner loop (mac_group) at full SM occupancy:
// every thread accumulates products of shared-memory rows for one column
// group, like phase A of the kernels. Prints executed limb-MACs per clock per SM.
#include <cstdio>
#include <cstdint>
#include "../paper_1908_09301_b200/csrc/mpt_device.cuh"
using namespace mpt;

template <int NT>
__global__ void __launch_bounds__(NT, 1) k(int W, int nrows, int reps, unsigned long long* out, long long* sink) {
  extern __shared__ int32_t rows[];
  const int rw = W + 2 * kPad + 1;
  for (int i = threadIdx.x; i < nrows * rw; i += NT) {
    const int d = i % rw - kPad;
    rows[i] = (d >= 0 && d < W) ? (int32_t)(((i * 2654435761u) >> 4) & 0x0fffffff) : 0;
  }
  __syncthreads();
  const int Lf = W - 1, T = Lf - 2, gf = T / kR, NG = (2 * Lf) / kR - gf + 1;
  const int ns = NT / NG;
  const int slot = threadIdx.x / NG, grp = threadIdx.x % NG;
  MacCount mc;
  Acc a0, a1;
  acc_zero(a0);
  acc_zero(a1);
  int c0v = 0, c1v = 0;
  long long t0 = clock64();
  if (slot < ns) {
    const int c0 = kR * (gf + grp);
    for (int r = 0; r < reps; r++)
      for (int kk = slot; kk < nrows / 3; kk += ns) {
        const int32_t* A = rows + (size_t)(3 * kk) * rw + kPad;
        const int32_t* B = rows + (size_t)(3 * kk + 1) * rw + kPad;
        const int32_t* C = rows + (size_t)(3 * kk + 2) * rw + kPad;
        mac_group(a0, c0v, A, make_int2(0, W - 1), B, make_int2(0, W - 1), c0, T, &mc);
        mac_group(a1, c1v, A, make_int2(0, W - 1), C, make_int2(0, W - 1), c0, T, &mc);
      }
  }
  __syncthreads();
  long long t1 = clock64();
  atomicAdd(&out[0], mc.executed);
  if (threadIdx.x == 0) atomicAdd(&out[1], (unsigned long long)(t1 - t0));
  if (a0.v[0] + a1.v[3] == 0x1234567) sink[0] = 1;
}

template <int NT>
void run(int W, int sms) {
  const int rw = W + 2 * kPad + 1;
  int nrows = (200 * 1024) / (4 * rw);
  nrows -= nrows % 3;
  size_t smem = (size_t)nrows * rw * 4;
  cudaFuncSetAttribute(k<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned long long* d;
  long long* s;
  cudaMalloc(&d, 16);
  cudaMalloc(&s, 8);
  cudaMemset(d, 0, 16);
  k<NT><<<sms, NT, smem>>>(W, nrows, 4, d, s);
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  printf("W=%4d threads=%4d rows=%3d : %.2f executed MACs/clk/SM  (%s)\n", W, NT, nrows,
         (double)h[0] / ((double)h[1] / sms) / sms, cudaGetErrorString(e));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int W : {62, 98, 264, 501}) {
    run<256>(W, sms);
    run<512>(W, sms);
    run<1024>(W, sms);
  }
  return 0;
}
