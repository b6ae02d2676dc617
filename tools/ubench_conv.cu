// MAC-pipe experiment (not part of the product): the digit convolution inner
// loop -- acc[r] += a[p] * b[c0 + r - p] over an 8-column register window, both
// operands streamed from shared memory, as in the kernels' Cauchy sums -- on
//   V0  the INT32 pipe : 28-bit digits, s64 += s32*s32 (IMAD.WIDE), no folds needed for 120 products
//   V1  the FP64 pipe  : 24-bit digits held as doubles, fma.rn.f64; products are 48 bits, so a
//                        column stays exact for 32 accumulations and is then folded (low 24
//                        bits stay, the rest moves one column up)
//   V2  INT8 tensor    : raw mma.sync.m16n8k32.s8 issue rate (what a Toeplitz/relaxed-product
//                        GEMM formulation of the Cauchy sums could use at best: 16 int8 MACs per
//                        28-bit digit product with 7-bit slices)
// Reported: digit products per second and bit^2 per second (digit products x digit bits^2), the
// quantity that compares formats. Run under ncu for the pipe counters:
//   ncu --metrics sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active ./ubench_conv
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int L = 512;        // digits per row
constexpr int THREADS = 256;  // 8 warps; thread t: window (t % 64) * 8 of the 512 low columns

__global__ void conv_imad(const int32_t* __restrict__ ga, const int32_t* __restrict__ gb, long long* out, int reps) {
  __shared__ int32_t A[L + 16], B[2 * L + 32];
  for (int i = threadIdx.x; i < L + 16; i += THREADS) A[i] = i < L ? ga[i] : 0;
  for (int i = threadIdx.x; i < 2 * L + 32; i += THREADS) B[i] = (i >= L && i < 2 * L) ? gb[i - L] : 0;
  __syncthreads();
  const int c0 = (threadIdx.x % 64) * 8, part = threadIdx.x / 64;  // 4 p-ranges of 128
  int64_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int rep = 0; rep < reps; rep++) {
    int32_t w[8];
#pragma unroll
    for (int r = 0; r < 8; r++) w[r] = B[L + c0 + r - part * 128];
#pragma unroll 4
    for (int p = part * 128; p < part * 128 + 128; p++) {
      const int32_t a = A[p], bn = B[L + c0 - p - 1];
#pragma unroll
      for (int r = 0; r < 8; r++) asm("mad.wide.s32 %0, %1, %2, %0;" : "+l"(acc[r]) : "r"(a), "r"(w[r]));
#pragma unroll
      for (int r = 7; r > 0; r--) w[r] = w[r - 1];
      w[0] = bn;
    }
#pragma unroll
    for (int r = 0; r < 8; r++) acc[r] >>= 7;  // keep the sums bounded across repetitions
  }
  long long s = 0;
  for (int r = 0; r < 8; r++) s += acc[r];
  if (s == 0x123456789abcLL) out[0] = s;
}

__global__ void conv_dfma(const int32_t* __restrict__ ga, const int32_t* __restrict__ gb, long long* out, int reps) {
  __shared__ double A[L + 16], B[2 * L + 32];
  for (int i = threadIdx.x; i < L + 16; i += THREADS) A[i] = i < L ? (double)(ga[i] >> 4) : 0.0;  // 24-bit digits
  for (int i = threadIdx.x; i < 2 * L + 32; i += THREADS) B[i] = (i >= L && i < 2 * L) ? (double)(gb[i - L] >> 4) : 0.0;
  __syncthreads();
  const int c0 = (threadIdx.x % 64) * 8, part = threadIdx.x / 64;
  double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  const double two24 = 16777216.0, inv24 = 1.0 / 16777216.0;
  for (int rep = 0; rep < reps; rep++) {
    double w[8];
#pragma unroll
    for (int r = 0; r < 8; r++) w[r] = B[L + c0 + r - part * 128];
    for (int p0 = part * 128; p0 < part * 128 + 128; p0 += 32) {
#pragma unroll 4
      for (int p = p0; p < p0 + 32; p++) {
        const double a = A[p], bn = B[L + c0 - p - 1];
#pragma unroll
        for (int r = 0; r < 8; r++) acc[r] = fma(a, w[r], acc[r]);
#pragma unroll
        for (int r = 7; r > 0; r--) w[r] = w[r - 1];
        w[0] = bn;
      }
      // exact fold after 32 accumulations of 48-bit products (< 2^53): carry = floor(acc / 2^24)
#pragma unroll
      for (int r = 0; r < 8; r++) {
        const double c = floor(acc[r] * inv24);
        acc[r] = fma(-c, two24, acc[r]);
        acc[r + 1] += c;
      }
    }
    acc[8] *= 0.5;
  }
  double s = 0;
  for (int r = 0; r < 9; r++) s += acc[r];
  if (s == 1234.5678) out[0] = 1;
}

__global__ void imma_raw(long long* out, int iters) {
  int c[8][4];
  for (int k = 0; k < 8; k++)
    for (int j = 0; j < 4; j++) c[k][j] = 0;
  int a0 = threadIdx.x, a1 = threadIdx.x * 3, a2 = threadIdx.x * 5, a3 = threadIdx.x * 7, b0 = threadIdx.x * 11, b1 = threadIdx.x * 13;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[k][0]), "+r"(c[k][1]), "+r"(c[k][2]), "+r"(c[k][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
  for (int k = 0; k < 8; k++)
    for (int j = 0; j < 4; j++) s += c[k][j];
  if (s == 0x7fffffff) out[1] = s;
}

template <typename F>
static float timed(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();  // warm-up
  cudaEventRecord(a);
  launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  int32_t h[L];
  for (int i = 0; i < L; i++) h[i] = (int32_t)(((i * 2654435761u) >> 4) & 0xfffffff) - (1 << 27);
  int32_t *da, *db;
  long long* dout;
  cudaMalloc(&da, sizeof h);
  cudaMalloc(&db, sizeof h);
  cudaMalloc(&dout, 64);
  cudaMemcpy(da, h, sizeof h, cudaMemcpyHostToDevice);
  cudaMemcpy(db, h, sizeof h, cudaMemcpyHostToDevice);
  const int reps = 200;
  for (int occ : {1, 2, 4}) {
    const int blocks = sms * occ;
    const double macs = (double)blocks * THREADS * reps * 128.0 * 8.0;
    const float m0 = timed([&] { conv_imad<<<blocks, THREADS>>>(da, db, dout, reps); });
    const float m1 = timed([&] { conv_dfma<<<blocks, THREADS>>>(da, db, dout, reps); });
    const double r0 = macs / (m0 * 1e-3), r1 = macs / (m1 * 1e-3);
    printf("{\"kernel\": \"window convolution, IMAD.WIDE, 28-bit digits\", \"ctas_per_sm\": %d, \"digit_macs_per_s\": %.4e, "
           "\"per_clk_per_sm\": %.2f, \"bit2_per_s\": %.4e}\n", occ, r0, r0 / (sms * (double)clk * 1e3), r0 * 784.0);
    printf("{\"kernel\": \"window convolution, DFMA, 24-bit digits, fold every 32\", \"ctas_per_sm\": %d, \"digit_macs_per_s\": %.4e, "
           "\"per_clk_per_sm\": %.2f, \"bit2_per_s\": %.4e}\n", occ, r1, r1 / (sms * (double)clk * 1e3), r1 * 576.0);
  }
  {
    const int blocks = sms * 4, iters = 4096;
    const float m2 = timed([&] { imma_raw<<<blocks, 256>>>(dout, iters); });
    const double ops = (double)blocks * 8 /*warps*/ * iters * 8.0 * (16.0 * 8.0 * 32.0);  // int8 MACs
    const double r2 = ops / (m2 * 1e-3);
    printf("{\"kernel\": \"mma.sync.m16n8k32.s8 raw issue\", \"int8_macs_per_s\": %.4e, \"per_clk_per_sm\": %.1f, "
           "\"digit_mac_equivalent_per_s\": %.4e, \"note\": \"16 int8 MACs per 28-bit digit product (7-bit slices), at 100%% tile use\"}\n",
           r2, r2 / (sms * (double)clk * 1e3), r2 / 16.0);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
