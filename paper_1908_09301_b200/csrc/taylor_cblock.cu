// Cluster-block kernel ("cblock"): one trajectory per thread-block cluster of
// G = 2..16 CTAs of 16 warps (sm_100a) -- single trajectories at medium
// precision (35..93 digits: configs[1], K = 500), where one SM cannot supply the
// digit products of an order fast enough and the rows still fit one SM's shared
// memory.
//
// Arithmetic: variant 3 (oracle/fixmodel.c jet_wp; reference taylor.py:117
// _jet_rows, reduction.py:149 convolve, taylor.py:168 horner_eval), the same as
// the warp and block kernels: every rounding is a function of the VALUE of an
// exact column sum, so the partition of the Cauchy sums over CTAs, warps and
// lanes cannot change a bit.
//
// Every CTA keeps every coefficient row in its own shared memory and computes
// the cheap, latency-critical part of an order REDUNDANTLY (assemble U_i, round,
// multiply by C_i, round the new row), so no row is ever published: the only
// exchange is an all-gather of partial Cauchy column sums (~1 KB per CTA and
// order) through distributed shared memory.
//
// Per order i:
//   P1   units: CTA g owns a contiguous block of k; its products (pair q, k) are
//        cut into balanced pairs of 4-column windows (h, H-1-h) of the top-aligned
//        NU-digit triangle (NU = Lf + 3 - min_k(z_{i-k} + z_k), zero digits
//        skipped; every unit costs 4 (NU+4) IMAD.WIDE). Warps alternate between the
//        pairs; a lane is (k slot, window pair), folds each window once, and the
//        k slots of a warp are summed with shuffles. Meanwhile the top warps
//        compute the non-integer linear product, stage C_i and the zero-digit
//        minimum of the next order's old terms.
//        Three side warps prepare everything of U^m that only needs row i
//        (constant, integer and non-integer linear terms) as pre[m].
//   P1b  column sums over this CTA's warps; every value is PUSHED into the receive
//        slot [i & 1][g] of every CTA (st.shared::cluster)
//   --   cluster barrier (release / acquire)
//   P3a  warp m: U^m = rndb(pre[m] + sum_q pm[q] sum_g recv[g][q])   (local reads)
//   P3b  U^m (x) C_i in chunks of 16 digits of U, one warp per (m, chunk): operands
//        in registers, fully unrolled
//   P3c  warp m: new row = rndb(sum of the chunk vectors), row sum
// The receive slots are double-buffered by the order's parity, so one cluster
// barrier per order suffices.
#include <cooperative_groups.h>

#include "taylor_warp_impl.cuh"

namespace cg = cooperative_groups;

namespace mpt {
namespace cb {

using wp::madw;
constexpr int kWarps = 16;
constexpr int kThreads = 32 * kWarps;
constexpr int kLo = 6;       // zero digits below digit 0 of every row (window reads reach -5)
constexpr int MC = 3;        // columns per lane of the target warps (Lf + 4 <= 96)
constexpr int DT = 3;        // variables, one target warp each
constexpr int kCols = 32 * MC;
constexpr int kMaxQ = 2;     // product pairs
constexpr int kUnit = 10;    // int64 per unit: two windows of 5 folded values
constexpr int kPC = 16;      // digits of U per chunk of the U (x) C_i product
constexpr int kCLo = 20;     // zero digits below digit 0 of the staged C_i
constexpr int kSumWarp0 = 8; // first warp of the P1b threads

struct Layout {
  int ncols, stride, nrows, bw, cw, sw, nbig, nE, h2p, nch, ustride;
  size_t off_rows, off_zt, off_cbuf, off_lbuf, off_ubuf, off_pre, off_nscr, off_st, off_scr, off_recv, total;
};

__host__ __device__ inline int pow2_ge(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

__host__ __device__ inline Layout make_layout(const Params& p, int G) {
  Layout L;
  L.ncols = p.Lf + 4;
  L.stride = (kLo + p.W) | 1;  // odd: lanes reading consecutive rows hit different banks
  L.nrows = p.D * (p.N + 1);
  L.bw = 4 + p.W + p.Lf + 4;
  L.cw = kCLo + 2 * p.Lf + 12;
  L.sw = p.W + 3;
  L.nbig = wp::n_big_lin(p);
  const int Hmax = (p.Lf + 3 + 3) / 4;
  L.nE = 4 * Hmax + 1;                 // elements (columns) of one pair's partial sums
  L.h2p = pow2_ge((Hmax + 1) / 2);     // lanes per k slot at the widest window
  L.nch = (p.W + kPC - 1) / kPC;
  L.ustride = kPC * L.nch + 4;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o += (bytes + 15) / 16 * 16;
    return r;
  };
  take(64);  // the operand prefetch of win_mac may read a few words below row 0
  L.off_rows = take(sizeof(int32_t) * ((size_t)L.nrows * L.stride + 2 * kLo));
  L.off_zt = take((size_t)L.nrows);
  L.off_cbuf = take(sizeof(int32_t) * (size_t)L.cw);
  L.off_lbuf = take(sizeof(int32_t) * (size_t)L.bw * (L.nbig > 0 ? L.nbig : 1));
  L.off_ubuf = take(sizeof(int32_t) * (size_t)DT * L.ustride);
  L.off_pre = take(sizeof(int64_t) * (size_t)DT * kCols);
  L.off_nscr = take(sizeof(int64_t) * (size_t)p.D * L.sw);
  L.off_st = take(sizeof(int32_t) * (size_t)p.D * p.RS + sizeof(int2) * kMaxD);
  // unit scratch [warp][window pair][10]; the chunk vectors of P3b reuse it
  const size_t scr1 = sizeof(int64_t) * (size_t)kWarps * L.h2p * kUnit;
  const size_t scr2 = sizeof(int64_t) * (size_t)DT * L.nch * kCols;
  L.off_scr = take(scr1 > scr2 ? scr1 : scr2);
  L.off_recv = take(sizeof(int64_t) * 2 * (size_t)G * kMaxQ * L.nE);
  L.total = o;
  return L;
}

// One 4-column window of a truncated product: elements r0 .. r0+3 of
// acc[u + v] += a'[u] b'[v] (a'[u] = ap[-u], b'[v] = bp[-v]; digits above the
// window tops are zero). Elements >= nu lie below the truncation and are
// dropped. o[0] += carry out of element r0 (belongs to element r0 - 1),
// o[1 + j] += element r0 + j after one fold.
__device__ __forceinline__ void win_mac(const int32_t* ap, const int32_t* bp, int r0, int nu, int64_t* o) {
  int64_t c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  const int32_t* bq = bp - r0;  // bq[u - j] = b'[r0 + j - u]
  int32_t b0 = bq[-3], b1 = bq[-2], b2 = bq[-1], b3;
  // operands of the next iteration are loaded before this iteration's products
  int32_t a0 = ap[0], a1 = ap[-1], a2 = ap[-2], a3 = ap[-3];
  int32_t n0 = bq[0], n1 = bq[1], n2 = bq[2], n3 = bq[3];
#pragma unroll 1
  for (int u = 0; u < r0 + 4; u += 4) {
    const int32_t x0 = a0, x1 = a1, x2 = a2, x3 = a3;
    const int32_t y0 = n0, y1 = n1, y2 = n2, y3 = n3;
    a0 = ap[-u - 4];
    a1 = ap[-u - 5];
    a2 = ap[-u - 6];
    a3 = ap[-u - 7];
    n0 = bq[u + 4];
    n1 = bq[u + 5];
    n2 = bq[u + 6];
    n3 = bq[u + 7];
    b3 = y0;
    c0 = madw(x0, b3, c0);
    c1 = madw(x0, b2, c1);
    c2 = madw(x0, b1, c2);
    c3 = madw(x0, b0, c3);
    b0 = y1;
    c0 = madw(x1, b0, c0);
    c1 = madw(x1, b3, c1);
    c2 = madw(x1, b2, c2);
    c3 = madw(x1, b1, c3);
    b1 = y2;
    c0 = madw(x2, b1, c0);
    c1 = madw(x2, b0, c1);
    c2 = madw(x2, b3, c2);
    c3 = madw(x2, b2, c3);
    b2 = y3;
    c0 = madw(x3, b2, c0);
    c1 = madw(x3, b1, c1);
    c2 = madw(x3, b0, c2);
    c3 = madw(x3, b3, c3);
  }
  if (r0 + 0 >= nu) c0 = 0;
  if (r0 + 1 >= nu) c1 = 0;
  if (r0 + 2 >= nu) c2 = 0;
  if (r0 + 3 >= nu) c3 = 0;
  o[0] += c0 >> kRadixBits;
  o[1] += (c0 & kMask) + (c1 >> kRadixBits);
  o[2] += (c1 & kMask) + (c2 >> kRadixBits);
  o[3] += (c2 & kMask) + (c3 >> kRadixBits);
  o[4] += c3 & kMask;
}

// one out-of-line copy of the rounding for all three call sites (instruction-cache
// footprint): columns lane*3 + j in, semi-normal digits (column - 2) of the exact value out
struct Sd3 {
  int32_t e0, e1, e2;
  int ovf;
};
__device__ __noinline__ Sd3 sd3(int64_t v0, int64_t v1, int64_t v2, int half, int Wout) {
  int64_t v[1][MC] = {{v0, v1, v2}};
  if (half && (threadIdx.x & 31) == 0) v[0][1] += kRadix / 2;  // column 1: the rounding half
  int32_t e[1][MC];
  const bool ovf = wp::warp_bal<MC, false, 1>(v, 1, Wout, e);
  Sd3 r;
  r.e0 = e[0][0];
  r.e1 = e[0][1];
  r.e2 = e[0][2];
  r.ovf = ovf;
  return r;
}

__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void st_remote64(uint32_t laddr, int rank, int64_t v) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(laddr), "r"(rank));
  asm volatile("st.shared::cluster.b64 [%0], %1;" ::"r"(ra), "l"(v) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1) taylor_cblock_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const unsigned full = 0xffffffffu;
  cg::cluster_group cluster = cg::this_cluster();
  const int G = (int)cluster.num_blocks(), g = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int traj = blockIdx.x / G;
  const Layout L = make_layout(p, G);
  int32_t* rows = (int32_t*)(smem + L.off_rows) + kLo;
  uint8_t* zt = (uint8_t*)(smem + L.off_zt);
  int32_t* cbuf = (int32_t*)(smem + L.off_cbuf) + kCLo;
  int32_t* lbuf = (int32_t*)(smem + L.off_lbuf) + 4;
  int32_t* ubuf = (int32_t*)(smem + L.off_ubuf);
  int64_t* pre = (int64_t*)(smem + L.off_pre);
  int64_t* nscr = (int64_t*)(smem + L.off_nscr);
  int32_t* st = (int32_t*)(smem + L.off_st);
  int2* stinfo = (int2*)(st + p.D * p.RS);
  int64_t* scr = (int64_t*)(smem + L.off_scr);
  int64_t* xpart = scr;  // P3b / P3c reuse the unit scratch
  int64_t* recv = (int64_t*)(smem + L.off_recv);
  __shared__ int s_ovf, s_zpre[2];
  const int D = p.D, N = p.N, N1 = p.N + 1, Lf = p.Lf, W = p.W, ncols = L.ncols, NP = p.NP;
  const int T = Lf - 2, Tc = Lf + p.sc - 2, stride = L.stride, nE = L.nE, rowlen = kMaxQ * L.nE;
  const int nch = L.nch, ustride = L.ustride;
  const float rG = 1.0f / (float)G;

  for (int w = tid; w < (int)(L.total / 4); w += kThreads) ((int32_t*)smem)[w] = 0;
  if (tid == 0) {
    s_ovf = 0;
    s_zpre[0] = s_zpre[1] = 255;
  }
  __syncthreads();
  int32_t* gstate = p.state + (size_t)traj * D * p.RS;
  for (int e = tid; e < D * p.RS; e += kThreads) st[e] = gstate[e];
  if (warp == 0) {
    int slot = 0;
    for (int e = 0; e < D * D; e++) {
      if (p.lin_small[e]) continue;
      for (int d = lane; d < W; d += 32) lbuf[slot * L.bw + d] = p.lin[(size_t)e * p.RS + d];
      slot++;
    }
  }
  __syncthreads();
  // every CTA has read the initial state before rank 0 can ever write the final one
  cluster_arrive();
  cluster_wait();

  // target role: warp m < D owns variable m (roundings)
  const int m = warp;
  const bool target = warp < D;
  int pm[kMaxQ];
#pragma unroll
  for (int q = 0; q < kMaxQ; q++) {
    int s = 0;
    for (int t = 0; t < p.NT; t++)
      if (target && p.tpair[t] == q && p.teq[t] == m) s += p.tq_int[t];
    pm[q] = s;
  }
  // side role (P1): warp 15 - e prepares pre[e] (everything of U^e that only needs row i);
  // warp 15 also stages C_i and the zero-digit minimum of the next order's old terms
  const int eq = (warp >= kWarps - D) ? kWarps - 1 - warp : -1;
  bool okc[MC];
  int32_t cstreg[MC];
  int linint[DT];
  unsigned bigmask = 0;
  int bigslot[DT];
#pragma unroll
  for (int j = 0; j < MC; j++) {
    const int c = lane * MC + j;
    okc[j] = c < ncols;
    const int d = c - 2;
    cstreg[j] = (eq >= 0 && d >= 0 && d < W) ? p.cst[(size_t)eq * p.RS + d] : 0;
  }
  {
    int slot = 0;
    for (int e = 0; e < D * D; e++) {
      const int mm = e / D, jv = e % D;
      const bool big = !p.lin_small[e];
#pragma unroll
      for (int t = 0; t < DT; t++)
        if (eq >= 0 && mm == eq && jv == t) {
          linint[t] = big ? 0 : p.lin_int[e];
          bigslot[t] = slot;
          if (big) bigmask |= 1u << t;
        }
      if (big) slot++;
    }
#pragma unroll
    for (int t = 0; t < DT; t++)
      if (eq < 0 || t >= D) {
        linint[t] = 0;
        bigslot[t] = 0;
      }
  }
  // unit role (P1): warps alternate between the pairs
  const int npd = NP > 0 ? NP : 1;
  const int uq = warp % npd, uwi = warp / npd;
  const int nwq = (kWarps - uq + npd - 1) / npd;  // warps of pair uq
  const int urowa = (NP > 0 ? p.pj[uq] : 0) * N1, urowb = (NP > 0 ? p.pk[uq] : 0) * N1;
  int zra[kMaxQ], zrb[kMaxQ];
#pragma unroll
  for (int q = 0; q < kMaxQ; q++) {
    zra[q] = q < NP ? p.pj[q] * N1 : 0;
    zrb[q] = q < NP ? p.pk[q] * N1 : 0;
  }
  // sum role (P1b): threads 256 .. 256 + NP * EH
  const int stid = tid - 32 * kSumWarp0;

  MacCount mcount;
  MacCount* mc = p.counters ? &mcount : nullptr;
  bool ovf = false;
  int64_t ssum[MC];  // target warps: running sum of the rows of variable m

  // development only (MPT_DEBUG): clock64 timestamps of rank 0, warps 0 / 8 / 13, first step
  const int dbg_w = warp == 0 ? 0 : warp == kSumWarp0 ? 1 : warp == kWarps - 3 ? 2 : -1;
  const bool dbg_on = p.dbg && g == 0 && lane == 0 && dbg_w >= 0 && traj == 0;
#define CB_TS(i_, k_)                                                                                       \
  do {                                                                                                      \
    if (dbg_on && n == p.start_step + 1 && (i_) < 256) p.dbg[((i_) * 3 + dbg_w) * 16 + (k_)] = clock64(); \
  } while (0)

  for (int n = p.start_step + 1; n <= p.n_steps; n++) {
    // ---- row 0 = sd(state), one variable per target warp
    if (target) {
      int64_t v[MC];
#pragma unroll
      for (int j = 0; j < MC; j++) {
        const int d = lane * MC + j - 2;
        v[j] = (d >= 0 && d < W) ? st[m * p.RS + d] : 0;
      }
      const Sd3 r = sd3(v[0], v[1], v[2], 0, W);
      ovf |= r.ovf != 0;
      const int32_t e0[MC] = {r.e0, r.e1, r.e2};
      const int z = wp::lead_zeros<MC>(e0, Lf);
#pragma unroll
      for (int j = 0; j < MC; j++) {
        const int d = lane * MC + j - 2;
        if (d >= 0 && d < W) rows[(m * N1) * stride + d] = e0[j];
        ssum[j] = e0[j];
      }
      if (lane == 0) zt[m * N1] = (uint8_t)z;
    }
    __syncthreads();

    for (int i = 0; i < N; i++) {
      CB_TS(i, 0);
      // ---- order-wide window: NU = Lf + 3 - min_k (z_{i-k} + z_k) over every pair;
      // the terms 0 < k < i were reduced during the previous order (s_zpre)
      int zmin = i >= 2 ? s_zpre[i & 1] : 255;
#pragma unroll
      for (int q = 0; q < kMaxQ; q++)
        if (q < NP) {
          zmin = min(zmin, (int)zt[zra[q] + i] + (int)zt[zrb[q]]);
          zmin = min(zmin, (int)zt[zra[q]] + (int)zt[zrb[q] + i]);
        }
      const int nu = NP > 0 ? Lf + 3 - zmin : 0, ctop = Lf + 2 - zmin;
      const int H = (nu + 3) >> 2, H2 = (H + 1) >> 1;
      const int EH = 4 * H + 1;                              // elements in flight this order (per pair)
      const int kblk = (int)(((float)(i + G) + 0.5f) * rG);  // ceil((i + 1) / G): k block of one CTA
      const int k0 = g * kblk, nk = max(0, min(kblk, i + 1 - k0));
      const int par = i & 1;
      const int h2p = H2 <= 1 ? 1 : H2 <= 2 ? 2 : H2 <= 4 ? 4 : H2 <= 8 ? 8 : 16;
      const int cw = 32 / h2p;  // k slots per warp
      CB_TS(i, 1);

      // ---- side warps: C_i, next order's zero-digit minimum, pre[eq]
      if (eq >= 0) {
        if (eq == 0) {
          for (int d = lane; d < W; d += 32) cbuf[d] = __ldg(p.ctab + (size_t)i * p.RS + d);
          // old terms of order i + 1: k = 1 .. i (rows <= i)
          int z = 255;
          for (int k = 1 + lane; k <= i; k += 32)
#pragma unroll
            for (int q = 0; q < kMaxQ; q++)
              if (q < NP) z = min(z, (int)zt[zra[q] + i + 1 - k] + (int)zt[zrb[q] + k]);
          z = __reduce_min_sync(full, z);
          if (lane == 0) s_zpre[(i + 1) & 1] = z;
        }
        if (eq < D) {
          int64_t x[MC];
#pragma unroll
          for (int j = 0; j < MC; j++) {
            const int d = lane * MC + j - 2;
            int64_t s = i == 0 ? (int64_t)cstreg[j] : 0;
            if (d >= 0 && d < W) {
#pragma unroll
              for (int t = 0; t < DT; t++)
                if (linint[t] != 0) s += (int64_t)linint[t] * rows[(t * N1 + i) * stride + d];
            }
            x[j] = s;
          }
          if (bigmask) {
#pragma unroll
            for (int t = 0; t < DT; t++) {
              if (bigmask & (1u << t)) {
                // tprod(lin[eq][t], a~_i^t): row digits broadcast from shared memory
                const int32_t* ar = rows + (t * N1 + i) * stride;
                const int wa = W - zt[t * N1 + i];  // digits above are zero
                const int32_t* lb[MC];
#pragma unroll
                for (int j = 0; j < MC; j++) lb[j] = lbuf + bigslot[t] * L.bw + (okc[j] ? lane * MC + j + T : -4);
#pragma unroll 4
                for (int pp = 0; pp < wa; pp++) {
                  const int32_t a = ar[pp];
#pragma unroll
                  for (int j = 0; j < MC; j++) x[j] = madw(a, lb[j][okc[j] ? -pp : 0], x[j]);
                }
                if (mc && g == 0) {
                  mc->executed += (unsigned long long)wa;
                  mc->useful += (unsigned long long)wa / 2 + 1;
                }
              }
            }
          }
#pragma unroll
          for (int j = 0; j < MC; j++) pre[eq * kCols + lane * MC + j] = x[j];
        }
      }
      CB_TS(i, 2);

      if (nu > 0) {
        // ---- P1: this CTA's share of the Cauchy sums; lane = (k slot, window pair)
        const int hp = lane & (h2p - 1), cs = lane / h2p;
        if (uwi * cw < nk && uq < NP) {
          int64_t o[kUnit];
#pragma unroll
          for (int t = 0; t < kUnit; t++) o[t] = 0;
          if (hp < H2) {
            const int h2 = H - 1 - hp;
            for (int kk = uwi * cw + cs; kk < nk; kk += nwq * cw) {
              const int k = k0 + kk;
              const int ra = urowa + i - k, rb = urowb + k;
              const int za = zt[ra], zb = zt[rb];
              const int sb = min(zb, zmin), sa = zmin - sb;
              const int32_t* ap = rows + ra * stride + Lf - sa;
              const int32_t* bp = rows + rb * stride + Lf - sb;
              win_mac(ap, bp, 4 * hp, nu, o);
              if (h2 != hp) win_mac(ap, bp, 4 * h2, nu, o + 5);
              if (mc) {
                mc->executed += 16ull * (hp + 1) + (h2 != hp ? 16ull * (h2 + 1) : 0ull);
                if (hp == 0) mc->useful += wp::useful_tri(nu, za - sa, zb - sb, Lf + 1 - za, Lf + 1 - zb);
              }
            }
          }
          CB_TS(i, 3);
          // sum the k slots of the warp
          for (int sft = h2p; sft < 32; sft <<= 1) {
#pragma unroll
            for (int t = 0; t < kUnit; t++) o[t] += __shfl_xor_sync(full, o[t], sft);
          }
          if (cs == 0 && hp < H2) {
            int64_t* dst = scr + (warp * L.h2p + hp) * kUnit;
#pragma unroll
            for (int t = 0; t < kUnit; t++) dst[t] = o[t];
          }
        }
        // sum threads: where this element's two contributions sit inside a warp's scratch
        int sq = 0, se = 0, o1 = -1, o2 = -1, nwa = 0;
        const bool summer = stid >= 0 && stid < NP * EH;
        if (summer) {
          sq = stid >= EH ? 1 : 0;
          se = stid - sq * EH;
          const int r = se - 1;
          nwa = min((kWarps - sq + npd - 1) / npd, (nk + cw - 1) / cw);  // active warps of pair sq
          if (r >= 0) {
            const int h = r >> 2;
            o1 = (h < H2 ? h : H - 1 - h) * kUnit + (h < H2 ? 0 : 5) + 1 + (r & 3);
          }
          if (((r + 1) & 3) == 0 && ((r + 1) >> 2) < H) {
            const int h = (r + 1) >> 2;
            o2 = (h < H2 ? h : H - 1 - h) * kUnit + (h < H2 ? 0 : 5);
          }
        }
        CB_TS(i, 4);
        __syncthreads();  // [S1] warp sums are in scratch
        // ---- P1b: element sums over the warps of a pair, pushed to every CTA's receive slot
        if (summer) {
          int64_t osum = 0;
          for (int wi = 0; wi < nwa; wi++) {
            const int64_t* base = scr + ((wi * npd + sq) * L.h2p) * kUnit;
            if (o1 >= 0) osum += base[o1];
            if (o2 >= 0) osum += base[o2];
          }
          const uint32_t la = smem_u32(recv + (par * G + g) * rowlen + sq * nE + se);
          for (int rk = 0; rk < G; rk++) st_remote64(la, rk, osum);
        }
        CB_TS(i, 5);
        cluster_arrive();
        cluster_wait();
      } else {
        __syncthreads();
      }
      CB_TS(i, 6);

      // ---- P3a: warp m assembles and rounds U^m
      if (target) {
        int64_t U[MC];
#pragma unroll
        for (int j = 0; j < MC; j++) U[j] = pre[m * kCols + lane * MC + j];
        if (nu > 0) {
#pragma unroll
          for (int q = 0; q < kMaxQ; q++) {
            if (pm[q] != 0) {
              int64_t acc[MC];
              const int64_t* src[MC];
#pragma unroll
              for (int j = 0; j < MC; j++) {
                const int r = ctop - (lane * MC + j);
                const bool ok = r >= -1 && r < nu;
                acc[j] = 0;
                // invalid columns read element 0 of an all-zero slot region (never pushed): offset nE - 1 + ...
                src[j] = ok ? recv + (par * G) * rowlen + q * nE + r + 1 : nullptr;
              }
#pragma unroll 4
              for (int rk = 0; rk < G; rk++) {
#pragma unroll
                for (int j = 0; j < MC; j++)
                  if (src[j]) acc[j] += src[j][rk * rowlen];
              }
#pragma unroll
              for (int j = 0; j < MC; j++) U[j] += (int64_t)pm[q] * acc[j];
            }
          }
        }
        CB_TS(i, 7);
        const Sd3 r = sd3(U[0], U[1], U[2], 1, W);
        ovf |= r.ovf != 0;
        const int32_t ureg[MC] = {r.e0, r.e1, r.e2};
        int32_t* ub = ubuf + m * ustride;
#pragma unroll
        for (int j = 0; j < MC; j++) {
          const int d = lane * MC + j - 2;
          if (d >= 0 && d < W) ub[d] = ureg[j];
        }
      }
      CB_TS(i, 9);
      __syncthreads();  // [S3] U digits

      // ---- P3b: U^m (x) C_i, one warp per (variable, chunk of 16 digits of U)
      for (int job = warp; job < D * nch; job += kWarps) {
        const int jm = job / nch, ch = job - jm * nch;
        const int p0 = ch * kPC;
        const int4* up = (const int4*)(ubuf + jm * ustride + p0);
        int32_t a[kPC];
#pragma unroll
        for (int t4 = 0; t4 < kPC / 4; t4++) {
          const int4 v = up[t4];
          a[4 * t4] = v.x;
          a[4 * t4 + 1] = v.y;
          a[4 * t4 + 2] = v.z;
          a[4 * t4 + 3] = v.w;
        }
        // x[j] = sum_t a[t] C[c_j + Tc - p0 - t], c_j = 3 lane + j: an 18-digit window of C_i
        const int32_t* cp = cbuf + lane * MC + Tc - p0 - (kPC - 1);
        int32_t cwin[kPC + MC - 1];
#pragma unroll
        for (int s2 = 0; s2 < kPC + MC - 1; s2++) cwin[s2] = cp[s2];
        int64_t x[MC];
#pragma unroll
        for (int j = 0; j < MC; j++) x[j] = 0;
#pragma unroll
        for (int t = 0; t < kPC; t++)
#pragma unroll
          for (int j = 0; j < MC; j++) x[j] = madw(a[t], cwin[kPC - 1 - t + j], x[j]);
#pragma unroll
        for (int j = 0; j < MC; j++) xpart[job * kCols + lane * MC + j] = okc[j] ? x[j] : 0;
        if (mc && g == 0) {
          mc->executed += (unsigned long long)kPC;
          mc->useful += (unsigned long long)kPC / 2 + 1;
        }
      }
      CB_TS(i, 11);
      __syncthreads();  // [S4] chunk vectors

      // ---- P3c: warp m rounds the new row
      if (target) {
        int64_t x[MC];
#pragma unroll
        for (int j = 0; j < MC; j++) x[j] = 0;
        for (int ch = 0; ch < nch; ch++) {
#pragma unroll
          for (int j = 0; j < MC; j++) x[j] += xpart[(m * nch + ch) * kCols + lane * MC + j];
        }
        const Sd3 r = sd3(x[0], x[1], x[2], 1, W);
        ovf |= r.ovf != 0;
        const int32_t rowreg[MC] = {r.e0, r.e1, r.e2};
        const int z2 = wp::lead_zeros<MC>(rowreg, Lf);
#pragma unroll
        for (int j = 0; j < MC; j++) {
          const int d = lane * MC + j - 2;
          if (d >= 0 && d < W) rows[(m * N1 + i + 1) * stride + d] = rowreg[j];
          ssum[j] += rowreg[j];
        }
        if (lane == 0) zt[m * N1 + i + 1] = (uint8_t)z2;
      }
      CB_TS(i, 13);
      __syncthreads();  // [S5] rows i+1 and their zero counts are visible
    }

    if (p.write_coef && g == 0) {
      int32_t* gcoef = p.coef + (size_t)traj * D * N1 * p.RS;
      // rows leave the kernel in canonical form: sd of the value the semi-normal digits hold
#pragma unroll 1
      for (int r = warp; r < D * N1; r += kWarps) {
        int64_t cv[1][MC];
        int32_t ce[1][MC];
#pragma unroll
        for (int j = 0; j < MC; j++) {
          const int d = lane * MC + j - 2;
          cv[0][j] = (d >= 0 && d < W) ? rows[r * stride + d] : 0;
        }
        wp::warp_sd<MC, false, 1>(cv, 1, W, ce);
#pragma unroll
        for (int j = 0; j < MC; j++) {
          const int d = lane * MC + j - 2;
          if (d >= 0 && d < p.RS) gcoef[(size_t)r * p.RS + d] = d < W ? ce[0][j] : 0;
        }
      }
    }
    // ---- state = RN_P(sum of the rows)
    if (target) {
#pragma unroll
      for (int j = 0; j < MC; j++) {
        const int d = lane * MC + j - 2;
        if (d >= 0 && d < L.sw) nscr[m * L.sw + d] = d < W ? ssum[j] : 0;
      }
      __syncwarp();
      ovf |= warp_normalize_small(nscr + m * L.sw, L.sw, 0, W, st + m * p.RS, &stinfo[m], p.P);
      __syncwarp();
      if (g == 0 && ((n % p.stride == 0) || (n == p.n_steps))) {
        const int slot = (n % p.stride == 0) ? (n / p.stride - p.start_step / p.stride)
                                             : (p.n_steps / p.stride - p.start_step / p.stride + 1);
        int32_t* dst = p.rec + ((size_t)slot * p.n_traj + traj) * D * p.RS + (size_t)m * p.RS;
        for (int d = lane; d < p.RS; d += 32) dst[d] = d < W ? st[m * p.RS + d] : 0;
      }
    }
    __syncthreads();
  }
  if (g == 0)
    for (int e = tid; e < D * p.RS; e += kThreads) gstate[e] = (e % p.RS) < W ? st[e] : 0;
  if (ovf && lane == 0) atomicOr(&s_ovf, 1);
  __syncthreads();
  if (tid == 0 && g == 0) p.status[traj] = s_ovf ? kOverflow : kOk;
  if (mc) {
    unsigned long long u = mcount.useful, xx = mcount.executed;
    for (int s = 16; s >= 1; s >>= 1) {
      u += __shfl_xor_sync(full, u, s);
      xx += __shfl_xor_sync(full, xx, s);
    }
    if (lane == 0) {
      atomicAdd(p.counters, u);
      atomicAdd(p.counters + 1, xx);
    }
  }
  // no CTA may exit while another can still write into its receive slots
  cluster_arrive();
  cluster_wait();
}

}  // namespace cb

bool cblock_supported(const Params& p) {
  return p.D <= cb::DT && p.all_q_small && p.NP >= 1 && p.NP <= cb::kMaxQ && p.Lf + 4 <= cb::kCols && p.Lf >= 3 &&
         p.N >= 1 && p.N + 1 <= 255 * 32;
}

size_t cblock_smem_bytes(const Params& p, int G) { return cb::make_layout(p, G).total; }

static cudaLaunchConfig_t cblock_cfg(const Params& p, int G, size_t smem, cudaStream_t stream, cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.n_traj * G);
  cfg.blockDim = dim3(cb::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

cudaError_t launch_cblock_kernel(const Params& p, int G, size_t smem, cudaStream_t stream) {
  const void* fn = (const void*)cb::taylor_cblock_kernel;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (G > 8) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = cblock_cfg(p, G, smem, stream, attr);
  Params pc = p;
  void* args[] = {&pc};
  return cudaLaunchKernelExC(&cfg, fn, args);
}

// clusters of G CTAs with this much shared memory that can be co-resident (0: none)
int cblock_max_clusters(const Params& p, size_t smem, int G) {
  const void* fn = (const void*)cb::taylor_cblock_kernel;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  if (G > 8 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchAttribute attr[1];
  Params one = p;
  one.n_traj = 1;
  cudaLaunchConfig_t cfg = cblock_cfg(one, G, smem, nullptr, attr);
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

}  // namespace mpt
