// Integer / FP64 pipe micro-benchmarks on B200 (sm_100a): which instruction
// form gives the most exact digit products per clock. Each thread runs 8
// independent accumulation chains; results are reported as operations per
// second for the whole device (CUDA events, after warm-up).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/ubench_int tools/ubench_int.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CHAINS 8

__device__ __forceinline__ int64_t mad_wide_s(int32_t a, int32_t b, int64_t c) {
  int64_t d;
  asm volatile("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t mad_wide_u(uint32_t a, uint32_t b, uint64_t c) {
  uint64_t d;
  asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}

template <int V>
__global__ void kern(int iters, const int32_t* __restrict__ in, long long* out) {
  const int tid = threadIdx.x + blockIdx.x * blockDim.x;
  int32_t x[CHAINS];
  for (int c = 0; c < CHAINS; c++) x[c] = in[(tid + c) & 1023];
  int32_t y = in[(tid * 7) & 1023];
  int64_t a64[CHAINS];
  uint32_t a32[CHAINS];
  double ad[CHAINS];
  for (int c = 0; c < CHAINS; c++) {
    a64[c] = c;
    a32[c] = c;
    ad[c] = c;
  }
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int32_t yy = __shfl_sync(0xffffffffu, y, u);  // non-uniform, cheap
#pragma unroll
      for (int c = 0; c < CHAINS; c++) {
        if (V == 0) a64[c] = mad_wide_s(x[c], yy, a64[c]);
        if (V == 1) a64[c] = (int64_t)mad_wide_u((uint32_t)x[c], (uint32_t)yy, (uint64_t)a64[c]);
        if (V == 2) asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(a32[c]) : "r"(x[c]), "r"(yy));  // IMAD
        if (V == 3) ad[c] = fma((double)x[c], (double)yy, ad[c]);      // DFMA (conversion hoisted?)
        if (V == 4) a64[c] += (int64_t)x[c] * (int64_t)yy;             // C++ form: fused IMAD.WIDE
      }
    }
    y += i;
  }
  long long s = 0;
  for (int c = 0; c < CHAINS; c++) s += a64[c] + a32[c] + (long long)ad[c];
  if (s == 0x7fffffffffffLL) out[0] = s;
}

template <int V>
double run(int sms, const int32_t* d_in, long long* d_out) {
  const int threads = 512, blocks = sms * 4, iters = 2048;
  kern<V><<<blocks, threads>>>(16, d_in, d_out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<V><<<blocks, threads>>>(iters, d_in, d_out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return (double)blocks * threads * iters * 8 * CHAINS / (ms * 1e-3);
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  int32_t* d_in;
  long long* d_out;
  cudaMalloc(&d_in, 4096 * 4);
  cudaMalloc(&d_out, 8);
  int32_t h[1024];
  for (int i = 0; i < 1024; i++) h[i] = (i * 2654435761u) >> 4;
  cudaMemcpy(d_in, h, sizeof h, cudaMemcpyHostToDevice);
  const char* names[] = {"mad.wide.s32 (s64 += s32*s32)", "mad.wide.u32 (u64 += u32*u32)",
                         "mad.lo.u32 (u32 += u32*u32)", "fma.rn.f64", "C++ s64 += (s64)s32*(s64)s32"};
  double r[5] = {run<0>(sms, d_in, d_out), run<1>(sms, d_in, d_out), run<2>(sms, d_in, d_out),
                 run<3>(sms, d_in, d_out), run<4>(sms, d_in, d_out)};
  printf("{\"sms\": %d, \"clock_khz\": %d, \"results\": [", sms, clk);
  for (int v = 0; v < 5; v++)
    printf("%s{\"op\": \"%s\", \"per_second\": %.4e, \"per_clk_per_sm\": %.2f}", v ? ", " : "", names[v], r[v],
           r[v] / (sms * (double)clk * 1e3));
  printf("]}\n");
  return 0;
}
