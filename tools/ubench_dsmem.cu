// DSMEM fan-out / fan-in bandwidth and signalling latency inside one 16-CTA
// cluster on B200 (not part of the product). Times with clock64 on rank 0
// and on the receivers.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

__device__ __forceinline__ void st_async_v4(uint32_t raddr, uint4 v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];"
               ::"r"(raddr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar) : "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, int rank) {
  uint32_t r; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank)); return r;
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, int bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, int par) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(b);
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(a), "r"(par) : "memory");
}

// mode 0: rank0 -> all others, generic remote stores (v4), bytes per target
// mode 1: rank0 -> all others, st.async with mbarrier completion
// mode 2: all others -> rank0 (fan-in), st.async
// mode 3: ping-pong latency rank0 <-> rank1 via st.async (one 16-B message)
__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(512, 1) k(int mode, int bytes, int reps, long long* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ uint64_t bar[2];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank(), tid = threadIdx.x;
  uint4* buf = (uint4*)sm;  // receive area: 16 slots of 8 KB
  if (tid == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  cl.sync();
  const uint32_t lbuf = (uint32_t)__cvta_generic_to_shared(buf), lbar = (uint32_t)__cvta_generic_to_shared(&bar[0]);
  long long t0 = clock64();
  int par = 0;
  for (int r = 0; r < reps; r++) {
    if (mode == 0 || mode == 1) {
      const int n16 = bytes / 16;
      if (rank != 0 && tid == 0) mbar_expect(&bar[0], mode == 1 ? bytes : 0);
      if (mode == 0) { if (rank != 0 && tid == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(lbar) : "memory"); }
      cl.sync();  // receivers armed
      if (rank == 0) {
        for (int w = tid; w < 15 * n16; w += 512) {
          const int dst = 1 + w / n16, j = w % n16;
          uint4 v = make_uint4(w, r, j, dst);
          if (mode == 0) {
            uint4* rp = cl.map_shared_rank(buf, dst);
            rp[j] = v;
          } else {
            st_async_v4(mapa(lbuf + 16 * j, dst), v, mapa(lbar, dst));
          }
        }
      }
      if (mode == 0) cl.sync(); else if (rank != 0) { mbar_wait(&bar[0], par); }
      par ^= 1;
      if (mode == 1) cl.sync();
    } else if (mode == 2) {
      const int n16 = bytes / 16;
      if (rank == 0 && tid == 0) mbar_expect(&bar[0], 15 * bytes);
      cl.sync();
      if (rank != 0)
        for (int j = tid; j < n16; j += 512)
          st_async_v4(mapa(lbuf + 16 * ((rank - 1) * n16 + j), 0), make_uint4(j, r, rank, 0), mapa(lbar, 0));
      if (rank == 0) mbar_wait(&bar[0], par);
      par ^= 1;
      cl.sync();
    } else if (mode == 3) {
      if (tid == 0 && rank <= 1) {
        mbar_expect(&bar[0], 16);
      }
      cl.sync();
      for (int q = 0; q < 100; q++) {
        if (tid == 0 && rank == 0) {
          st_async_v4(mapa(lbuf, 1), make_uint4(q, 0, 0, 0), mapa(lbar, 1));
          mbar_wait(&bar[0], q & 1);
          mbar_expect(&bar[0], 16);
        }
        if (tid == 0 && rank == 1) {
          mbar_wait(&bar[0], q & 1);
          mbar_expect(&bar[0], 16);
          st_async_v4(mapa(lbuf, 0), make_uint4(q, 0, 0, 0), mapa(lbar, 0));
        }
      }
      break;
    }
  }
  long long t1 = clock64();
  if (tid == 0 && rank == 0) out[0] = t1 - t0;
  cl.sync();
}

int main() {
  long long* d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  const int reps = 200;
  // baseline: barriers only
  for (int mode : {0, 1, 2}) {
    for (int bytes : {16, 256, 1024, 4096}) {
      k<<<16, 512, 140 * 1024>>>(mode, bytes, reps, d);
      long long h; cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("{\"mode\": %d, \"bytes_per_peer\": %d, \"cycles_per_rep\": %.1f, \"total_bytes\": %d, \"err\": \"%s\"}\n",
             mode, bytes, (double)h / reps, 15 * bytes, cudaGetErrorString(e));
    }
  }
  k<<<16, 512, 140 * 1024>>>(3, 16, 1, d);
  long long h; cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("{\"mode\": 3, \"round_trip_cycles\": %.1f, \"err\": \"%s\"}\n", h / 100.0, cudaGetErrorString(e));
  return 0;
}
