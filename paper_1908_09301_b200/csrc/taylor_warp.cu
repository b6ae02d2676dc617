// Warp kernel, one column per lane (Lf + 4 <= 32), and its host side.
// See taylor_warp_impl.cuh for the algorithm.
#include "taylor_warp_impl.cuh"

namespace mpt {

const void* warp_fn_mc2(const Params& p);  // taylor_warp2.cu: two columns per lane

bool warp_supported(const Params& p) {
  const int gl = (p.D <= 3 && p.NP <= 2) ? 16 : 8;  // lanes per pair (warp_fn_mc)
  const int passes = (p.N + gl) / gl;               // products one lane accumulates per order
  // passes x NU digit products of at most (2^27 + 1)^2 each (semi-normal digits) in one int64 column (< 2^63)
  return p.D <= kMaxD && p.all_q_small && p.NP <= wp::kMaxPairs && p.Lf + 3 <= wp::kMaxNU && p.Lf >= 3 &&
         passes * (p.Lf + 3) <= 500 && p.W <= 64;
}

size_t warp_traj_smem(const Params& p) { return wp::make_layout(p).total; }

static const void* warp_fn(const Params& p) {
  return p.Lf + 4 > 32 ? warp_fn_mc2(p) : wp::warp_fn_mc<1>(p);
}

// warps (trajectories) per CTA that fit the most warps on one SM: smem_sm = shared
// memory per SM, optin = per-CTA limit
int warp_choose_wpb(const Params& p, size_t smem_sm, size_t optin) {
  const size_t per = warp_traj_smem(p);
  int best = 0, best_warps = 0;
  for (int wpb = 1; wpb <= 4; wpb++) {
    const size_t cta = per * wpb;
    if (cta > optin) break;
    int ctas = (int)(smem_sm / (cta + 1024));
    if (ctas > 32) ctas = 32;
    int warps = ctas * wpb;
    if (warps > 48) warps = 48;
    if (warps >= best_warps && warps > 0) {
      best_warps = warps;
      best = wpb;
    }
  }
  return best;
}

cudaError_t launch_warp_kernel(const Params& p, int wpb, cudaStream_t stream) {
  const void* fn = warp_fn(p);
  const size_t smem = warp_traj_smem(p) * wpb;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int blocks = (p.n_traj + wpb - 1) / wpb;
  Params pp = p;
  void* args[] = {(void*)&pp};
  return cudaLaunchKernel(fn, dim3(blocks), dim3(32 * wpb), args, smem, stream);
}

}  // namespace mpt
