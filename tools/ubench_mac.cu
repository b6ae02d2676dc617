// Digit-product throughput probes on one B200 (not part of the product):
//   V0: s64 += (s64)s32*s32            (IMAD.WIDE + IADD3 pairs)
//   V1: f64 = fma(f64, f64, f64)       (DFMA, operands already double)
//   V2: half the chains V0, half V1     (INT and FP64 pipes together)
// plus the dependent-chain latency of each op.
#include <cstdio>
#include <cstdint>
#define CH 8
template <int V>
__global__ void thr(int iters, const double* __restrict__ in, long long* out) {
  const int tid = threadIdx.x + blockIdx.x * blockDim.x;
  int32_t xi[CH]; double xd[CH]; int64_t ai[CH]; double ad[CH];
  for (int c = 0; c < CH; c++) { xd[c] = in[(tid + c) & 1023]; xi[c] = (int32_t)xd[c]; ai[c] = c; ad[c] = c; }
  double yd = in[(tid * 7) & 1023]; int32_t yi = (int32_t)yd;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const double y1 = __shfl_sync(0xffffffffu, yd, u);
      const int32_t y2 = __shfl_sync(0xffffffffu, yi, u);
#pragma unroll
      for (int c = 0; c < CH; c++) {
        if (V == 0 || (V == 2 && c < CH / 2)) ai[c] += (int64_t)xi[c] * (int64_t)y2;
        if (V == 1 || (V == 2 && c >= CH / 2)) ad[c] = fma(xd[c], y1, ad[c]);
      }
    }
    yd += 1.0; yi += i;
  }
  double s = 0;
  for (int c = 0; c < CH; c++) s += (double)ai[c] + ad[c];
  if (s == 12345.678) out[0] = 1;
}
template <int V>
__global__ void lat(int iters, const double* __restrict__ in, long long* out) {
  double d = in[threadIdx.x], e = in[threadIdx.x + 1];
  int64_t a = (int64_t)d; int32_t x = (int32_t)e;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
    if (V == 0) a += (int64_t)(int32_t)a * (int64_t)x;
    if (V == 1) d = fma(d, e, d);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[V] = (t1 - t0);
  if (a + d == 1234.5) out[3] = 1;
}
template <int V>
double run(int sms, const double* d_in, long long* d_out, int blocks_per_sm, int threads) {
  const int blocks = sms * blocks_per_sm, iters = 4096;
  thr<V><<<blocks, threads>>>(16, d_in, d_out);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  thr<V><<<blocks, threads>>>(iters, d_in, d_out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return (double)blocks * threads * iters * 8 * CH / (ms * 1e-3);
}
int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d_in; long long* d_out;
  cudaMalloc(&d_in, 4096 * 8); cudaMalloc(&d_out, 64);
  double h[1024];
  for (int i = 0; i < 1024; i++) h[i] = (double)(((i * 2654435761u) >> 8) & 0xffffff) - 8388608.0;
  cudaMemcpy(d_in, h, sizeof h, cudaMemcpyHostToDevice);
  const char* names[] = {"s64 += s32*s32 (IMAD.WIDE)", "fma.rn.f64 (DFMA)", "half IMAD.WIDE + half DFMA"};
  for (int occ : {1, 2, 4}) {
    double r[3] = {run<0>(sms, d_in, d_out, occ, 512), run<1>(sms, d_in, d_out, occ, 512), run<2>(sms, d_in, d_out, occ, 512)};
    for (int v = 0; v < 3; v++)
      printf("{\"op\": \"%s\", \"ctas_per_sm\": %d, \"threads\": 512, \"per_second\": %.4e, \"per_clk_per_sm\": %.2f}\n",
             names[v], occ, r[v], r[v] / (sms * (double)clk * 1e3));
  }
  lat<0><<<1, 32>>>(1000, d_in, d_out); lat<1><<<1, 32>>>(1000, d_in, d_out);
  long long hl[2]; cudaMemcpy(hl, d_out, 16, cudaMemcpyDeviceToHost);
  printf("{\"latency_cycles\": {\"imad_wide_chain\": %.2f, \"dfma_chain\": %.2f}}\n", hl[0] / 1000.0, hl[1] / 1000.0);
  return 0;
}
