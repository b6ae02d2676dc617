// Block kernel ("block"): one trajectory per CTA of 8 warps, coefficient rows
// resident in shared memory -- ensembles at medium precision (35..58 digits:
// configs[4] at K = 400 and its K = 450 verify runs), where the rows of one
// trajectory fill most of an SM's shared memory.
//
// Same arithmetic as the warp kernel (oracle/fixmodel.c jet_wp, variant 3:
// value-exact roundings (kept in semi-normal digits inside the kernel, canonical sd digits on output), direct per-order recurrence; reference
// taylor.py:117 _jet_rows, reduction.py:149 convolve, taylor.py:168
// horner_eval) and the same building blocks (taylor_warp_impl.cuh): top-aligned
// NU-digit windows, a fully unrolled register triangle per lane, one fold, a
// shuffle reduce-scatter per warp. What changes is the width: four warps per
// product pair take k = l, l + 128, ...; each warp leaves its reduced columns
// in shared memory; after one CTA barrier warp m assembles U^m from the four
// partial column vectors of every pair and rounds it; U^m (x) C_i is cut into
// chunks of 32 digits of U, one warp per (variable, chunk), operands in registers;
// warp m sums the chunk vectors and rounds the new row. Four CTA barriers per order.
#include "taylor_warp_impl.cuh"

namespace mpt {
namespace blk {

using wp::kLo;
using wp::madw;
constexpr int kWarps = 8;
constexpr int kThreads = 32 * kWarps;
constexpr int kMaxNU = 60;   // Lf + 3 <= 60
constexpr int MC = 2;        // columns per lane (Lf + 4 <= 64)
constexpr int DT = 3;        // variables, one target warp each
constexpr int kPairWarps = 4;
constexpr int kPartCols = 68;  // 64 reduced columns + the carry out of the top one
constexpr int kPC = 32;        // digits of U per chunk of the U (x) C_i product (one warp per variable and chunk)
constexpr int kCLo = 36;       // zero digits below digit 0 of the staged C_i
constexpr int kCols = 32 * MC;

struct Layout {
  int ncols, stride, nrows, bw, sw, nbig, nch, ustride;
  size_t off_rows, off_zt, off_bbuf, off_lbuf, off_ubuf, off_part, off_xpart, off_lpart, off_scr, off_st, total;
};

__host__ __device__ inline Layout make_layout(const Params& p) {
  Layout L;
  L.ncols = p.Lf + 4;
  L.stride = (kLo + p.W) | 1;
  L.nrows = p.D * (p.N + 1);
  L.bw = kCLo + p.W + p.Lf + 8;  // zero-padded constant operand of the chunked products
  L.sw = p.W + 3;
  L.nbig = wp::n_big_lin(p);
  L.nch = (p.W + kPC - 1) / kPC;
  L.ustride = kPC * L.nch + 4;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o += (bytes + 15) / 16 * 16;
    return r;
  };
  L.off_rows = take(sizeof(int32_t) * ((size_t)L.nrows * L.stride + 2 * kLo));
  L.off_zt = take((size_t)L.nrows);
  L.off_bbuf = take(sizeof(int32_t) * (size_t)L.bw);
  L.off_lbuf = take(sizeof(int32_t) * (size_t)L.bw * L.nbig);
  L.off_ubuf = take(sizeof(int32_t) * (size_t)DT * L.ustride);
  L.off_part = take(sizeof(int64_t) * 2 * kPairWarps * kPartCols);
  L.off_xpart = take(sizeof(int64_t) * (size_t)DT * L.nch * kCols);
  L.off_lpart = take(sizeof(int64_t) * (size_t)(L.nbig > 0 ? DT * L.nch * kCols : 0));
  L.off_scr = take(sizeof(int64_t) * (size_t)p.D * L.sw);
  L.off_st = take(sizeof(int32_t) * (size_t)p.D * p.RS + sizeof(int2) * kMaxD);
  L.total = o;
  return L;
}

// acc[u + v] += a'[u] b'[v], u + v < NU; b' held in registers, a' streamed
template <int NU>
__device__ __forceinline__ void tri_mac_s(int64_t (&acc)[NU], const int32_t* ap, const int32_t* bp) {
  int32_t b[NU];
#pragma unroll
  for (int v = 0; v < NU; v++) b[v] = bp[-v];
#pragma unroll
  for (int u = 0; u < NU; u++) {
    const int32_t a = ap[-u];
#pragma unroll
    for (int v = 0; v + u < NU; v++) acc[u + v] = madw(a, b[v], acc[u + v]);
  }
}

// One warp's share of the Cauchy sum of its pair: k = kl, kl + 128, ...; the
// reduced columns (element r = column ctop - r) go to out[0..NP2), the carry
// out of the top column to out[kPartCols - 1].
template <int NU>
__device__ __forceinline__ void cauchy_part(const wp::Ctx& cx, int va, int vb, int i, int zmin, int kl,
                                            int64_t* out, MacCount* mc) {
  constexpr int NP2 = NU <= 4 ? 4 : NU <= 8 ? 8 : NU <= 16 ? 16 : NU <= 32 ? 32 : 64;
  constexpr int E = NP2 >= 32 ? NP2 / 32 : 1;
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int nureal = cx.Lf + 3 - zmin;
  int64_t acc[NU];
#pragma unroll
  for (int r = 0; r < NU; r++) acc[r] = 0;
  for (int k = kl; k <= i; k += 32 * kPairWarps) {
    const int ra = va * cx.N1 + i - k, rb = vb * cx.N1 + k;
    const int za = cx.zt[ra], zb = cx.zt[rb];
    const int sb = min(zb, zmin), sa = zmin - sb;
    tri_mac_s<NU>(acc, cx.rows + (size_t)ra * cx.stride + cx.Lf - sa, cx.rows + (size_t)rb * cx.stride + cx.Lf - sb);
    if (mc) {
      mc->useful += wp::useful_tri(nureal, za - sa, zb - sb, cx.Lf + 1 - za, cx.Lf + 1 - zb);
      mc->executed += NU * (NU + 1) / 2;
    }
  }
  __syncwarp();
#pragma unroll
  for (int r = (NU >= 3 ? NU - 3 : 0); r < NU; r++)
    if (r >= nureal) acc[r] = 0;
  int64_t v[NP2];
  int64_t x = acc[0] >> kRadixBits;
#pragma unroll
  for (int r = 0; r < NP2; r++) {
    if (r < NU)
      v[r] = (acc[r] & kMask) + (r + 1 < NU ? (acc[r + 1] >> kRadixBits) : 0);
    else
      v[r] = 0;
  }
  int n = NP2;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    if (n > 1) {
      const int half = n / 2;
      const bool up = (lane & s) != 0;
#pragma unroll
      for (int j = 0; j < NP2 / 2; j++) {
        if (j < half) {
          const int64_t send = up ? v[j] : v[half + j];
          const int64_t keep = up ? v[half + j] : v[j];
          v[j] = keep + __shfl_xor_sync(full, send, s);
        }
      }
      n = half;
    } else {
      v[0] += __shfl_xor_sync(full, v[0], s);
    }
    x += __shfl_xor_sync(full, x, s);
  }
  if (NP2 >= 32) {
#pragma unroll
    for (int ee = 0; ee < E; ee++) out[lane * E + ee] = v[ee];
  } else {
    if (lane % (32 / (NP2 >= 32 ? 32 : NP2)) == 0) out[lane / (32 / (NP2 >= 32 ? 32 : NP2))] = v[0];
  }
  if (lane == 0) out[kPartCols - 1] = x;
}

__device__ __forceinline__ void cauchy_dispatch(const wp::Ctx& cx, int va, int vb, int i, int zmin, int kl, int64_t* out,
                                                MacCount* mc) {
  const int nureal = cx.Lf + 3 - zmin;
  switch ((nureal + 3) >> 2) {
    case 1: cauchy_part<4>(cx, va, vb, i, zmin, kl, out, mc); break;
    case 2: cauchy_part<8>(cx, va, vb, i, zmin, kl, out, mc); break;
    case 3: cauchy_part<12>(cx, va, vb, i, zmin, kl, out, mc); break;
    case 4: cauchy_part<16>(cx, va, vb, i, zmin, kl, out, mc); break;
    case 5: cauchy_part<20>(cx, va, vb, i, zmin, kl, out, mc); break;
    case 6: cauchy_part<24>(cx, va, vb, i, zmin, kl, out, mc); break;
    case 7: cauchy_part<28>(cx, va, vb, i, zmin, kl, out, mc); break;
    case 8: cauchy_part<32>(cx, va, vb, i, zmin, kl, out, mc); break;
    case 9: cauchy_part<36>(cx, va, vb, i, zmin, kl, out, mc); break;
    case 10: cauchy_part<40>(cx, va, vb, i, zmin, kl, out, mc); break;
    case 11: cauchy_part<44>(cx, va, vb, i, zmin, kl, out, mc); break;
    case 12: cauchy_part<48>(cx, va, vb, i, zmin, kl, out, mc); break;
    case 13: cauchy_part<52>(cx, va, vb, i, zmin, kl, out, mc); break;
    case 14: cauchy_part<56>(cx, va, vb, i, zmin, kl, out, mc); break;
    default: cauchy_part<kMaxNU>(cx, va, vb, i, zmin, kl, out, mc); break;
  }
}

__global__ void __launch_bounds__(kThreads, 1) taylor_block_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const unsigned full = 0xffffffffu;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int traj = blockIdx.x;
  const Layout L = make_layout(p);
  int32_t* rows = (int32_t*)(smem + L.off_rows) + kLo;
  uint8_t* zt = (uint8_t*)(smem + L.off_zt);
  int32_t* bbuf = (int32_t*)(smem + L.off_bbuf) + kCLo;
  int32_t* lbuf = (int32_t*)(smem + L.off_lbuf) + kCLo;
  int32_t* ubuf = (int32_t*)(smem + L.off_ubuf);
  int64_t* part = (int64_t*)(smem + L.off_part);
  int64_t* xpart = (int64_t*)(smem + L.off_xpart);
  int64_t* lpart = (int64_t*)(smem + L.off_lpart);
  int64_t* scr = (int64_t*)(smem + L.off_scr);
  int32_t* st = (int32_t*)(smem + L.off_st);
  int2* stinfo = (int2*)(st + (size_t)p.D * p.RS);
  __shared__ int s_ovf;
  const int D = p.D, N = p.N, N1 = p.N + 1, Lf = p.Lf, W = p.W, ncols = L.ncols;
  const int T = Lf - 2, Tc = Lf + p.sc - 2;

  for (size_t w = tid; w < L.total / 4; w += kThreads) ((int32_t*)smem)[w] = 0;
  if (tid == 0) s_ovf = 0;
  __syncthreads();
  int32_t* gstate = p.state + (size_t)traj * D * p.RS;
  for (int e = tid; e < D * p.RS; e += kThreads) st[e] = gstate[e];
  if (warp == 0) {
    int slot = 0;
    for (int e = 0; e < D * D; e++) {
      if (p.lin_small[e]) continue;
      for (int d = lane; d < W; d += 32) lbuf[(size_t)slot * L.bw + d] = p.lin[(size_t)e * p.RS + d];
      slot++;
    }
  }
  __syncthreads();

  // Cauchy role: warps 0..3 -> pair 0, warps 4..7 -> pair 1; lane's first k
  const int pq = warp / kPairWarps, kl = (warp % kPairWarps) * 32 + lane;
  const int va = pq < p.NP ? p.pj[pq] : 0, vb = pq < p.NP ? p.pk[pq] : 0;
  // target role: warp m < D owns variable m
  const int m = warp;
  const bool target = warp < D;
  bool okc[MC];
  int32_t cstreg[MC];
  int pm[2], linint[DT];
  unsigned bigmask = 0;  // bit jv: lin[m][jv] needs a full product
  int bigslot[DT];
#pragma unroll
  for (int j = 0; j < MC; j++) {
    const int c = lane * MC + j;
    okc[j] = c < ncols;
    const int d = c - 2;
    cstreg[j] = (target && d >= 0 && d < W) ? p.cst[(size_t)m * p.RS + d] : 0;
  }
#pragma unroll
  for (int q = 0; q < 2; q++) {
    int s = 0;
    for (int t = 0; t < p.NT; t++)
      if (target && p.tpair[t] == q && p.teq[t] == m) s += p.tq_int[t];
    pm[q] = s;
  }
  {
    int slot = 0;
    for (int e = 0; e < D * D; e++) {
      const int mm = e / D, jv = e % D;
      const bool big = !p.lin_small[e];
#pragma unroll
      for (int t = 0; t < DT; t++)
        if (target && mm == m && jv == t) {
          linint[t] = big ? 0 : p.lin_int[e];
          bigslot[t] = slot;
          if (big) bigmask |= 1u << t;
        }
      if (big) slot++;
    }
#pragma unroll
    for (int t = 0; t < DT; t++)
      if (!target || t >= D) {
        linint[t] = 0;
        bigslot[t] = 0;
      }
  }

  // linear-product role (phase 1): warp 7 - job computes one 32-digit chunk of the non-integer
  // linear products of one equation (D equations x nch <= 2 chunks <= 6 jobs)
  int job_m = -1, job_ch = 0;
  unsigned jobmask = 0;
  int jobslot[DT];
  {
    const int jw = kWarps - 1 - warp;
    int nb = 0;
    for (int mm = 0; mm < D; mm++) {
      bool big = false;
      for (int t = 0; t < D; t++) big |= !p.lin_small[mm * D + t];
      if (big) {
        if (jw / L.nch == nb) {
          job_m = mm;
          job_ch = jw % L.nch;
        }
        nb++;
      }
    }
    int slot = 0;
    for (int e = 0; e < D * D; e++) {
      if (p.lin_small[e]) continue;
#pragma unroll
      for (int t = 0; t < DT; t++)
        if (job_m >= 0 && e / D == job_m && e % D == t) {
          jobmask |= 1u << t;
          jobslot[t] = slot;
        }
      slot++;
    }
#pragma unroll
    for (int t = 0; t < DT; t++)
      if (!(jobmask & (1u << t))) jobslot[t] = 0;
  }

  wp::Ctx cx{rows, zt, L.stride, N1, Lf, p.NP};
  MacCount mcount;
  MacCount* mc = p.counters ? &mcount : nullptr;
  bool ovf = false;
  int64_t ssum[MC];  // target warps: running sum of the rows of variable m

  for (int n = p.start_step + 1; n <= p.n_steps; n++) {
    // ---- row 0 = sd(state), one variable per target warp
    if (target) {
      int64_t v[1][MC];
      int32_t e0[1][MC];
#pragma unroll
      for (int j = 0; j < MC; j++) {
        const int d = lane * MC + j - 2;
        v[0][j] = (d >= 0 && d < W) ? st[m * p.RS + d] : 0;
      }
      ovf |= wp::warp_bal<MC, false, 1>(v, 1, W, e0);
      const int z = wp::lead_zeros<MC>(e0[0], Lf);
#pragma unroll
      for (int j = 0; j < MC; j++) {
        const int d = lane * MC + j - 2;
        if (d >= 0 && d < W) rows[(size_t)(m * N1) * L.stride + d] = e0[0][j];
        ssum[j] = e0[0][j];
      }
      if (lane == 0) zt[m * N1] = (uint8_t)z;
    }
    __syncthreads();

    for (int i = 0; i < N; i++) {
      // ---- phase 1: every warp its share of its pair's Cauchy sum
      int z = 255;
      for (int k = lane; k <= i; k += 32)
#pragma unroll
        for (int q = 0; q < 2; q++)
          if (q < p.NP) z = min(z, (int)zt[p.pj[q] * N1 + i - k] + (int)zt[p.pk[q] * N1 + k]);
      const int zmin = __reduce_min_sync(full, z);
      const int nureal = Lf + 3 - zmin, ctop = Lf + 2 - zmin;
      if (job_m >= 0) {
        // tprod(lin[job_m][t], a~_i^t), digits p0 .. p0+31 of the row: operands in registers
        const int p0 = job_ch * kPC;
        int64_t x[MC];
#pragma unroll
        for (int j = 0; j < MC; j++) x[j] = 0;
#pragma unroll
        for (int t = 0; t < DT; t++) {
          if (jobmask & (1u << t)) {
            const int32_t* ar = rows + (size_t)(t * N1 + i) * L.stride + p0;
            int32_t a[kPC];
#pragma unroll
            for (int tt = 0; tt < kPC; tt++) a[tt] = p0 + tt < W ? ar[tt] : 0;
            const int32_t* cp = lbuf + (size_t)jobslot[t] * L.bw + lane * MC + T - p0 - (kPC - 1);
            int32_t cwin[kPC + MC - 1];
#pragma unroll
            for (int s2 = 0; s2 < kPC + MC - 1; s2++) cwin[s2] = cp[s2];
#pragma unroll
            for (int tt = 0; tt < kPC; tt++)
#pragma unroll
              for (int j = 0; j < MC; j++) x[j] = madw(a[tt], cwin[kPC - 1 - tt + j], x[j]);
            if (mc) {
              mc->executed += (unsigned long long)kPC;
              mc->useful += (unsigned long long)kPC / 2 + 1;
            }
          }
        }
#pragma unroll
        for (int j = 0; j < MC; j++) lpart[(size_t)(job_m * L.nch + job_ch) * kCols + lane * MC + j] = okc[j] ? x[j] : 0;
      }
      if (pq < p.NP && nureal > 0)
        cauchy_dispatch(cx, va, vb, i, zmin, kl, part + (size_t)warp * kPartCols, mc);
      if (warp == kWarps - 1) {  // C_i into the padded operand buffer
        for (int d = lane; d < W; d += 32) bbuf[d] = __ldg(p.ctab + (size_t)i * p.RS + d);
      }
      __syncthreads();  // [A] partial columns and C_i are in shared memory

      // ---- phase 2: warp m assembles U^m, rounds, multiplies by C_i, rounds the new row
      if (target) {
        int64_t U[1][MC];
#pragma unroll
        for (int j = 0; j < MC; j++) {
          const int c = lane * MC + j, d = c - 2;
          int64_t s = i == 0 ? (int64_t)cstreg[j] : 0;
          if (d >= 0 && d < W) {
#pragma unroll
            for (int t = 0; t < DT; t++)
              if (linint[t] != 0) s += (int64_t)linint[t] * rows[(size_t)(t * N1 + i) * L.stride + d];
          }
          if (nureal > 0) {
            const int r = ctop - c;
#pragma unroll
            for (int q = 0; q < 2; q++) {
              if (pm[q] != 0) {
                int64_t cs = 0;
                if (r >= -1 && r < nureal) {
                  const int64_t* pp = part + (size_t)(q * kPairWarps) * kPartCols + (r >= 0 ? r : kPartCols - 1);
#pragma unroll
                  for (int w4 = 0; w4 < kPairWarps; w4++) cs += pp[(size_t)w4 * kPartCols];
                }
                s += (int64_t)pm[q] * cs;
              }
            }
          }
          U[0][j] = s;
        }
        if (bigmask) {  // the chunk vectors of the non-integer linear products (phase 1)
          for (int ch = 0; ch < L.nch; ch++) {
#pragma unroll
            for (int j = 0; j < MC; j++) U[0][j] += lpart[(size_t)(m * L.nch + ch) * kCols + lane * MC + j];
          }
        }
        int32_t ureg[1][MC];
        ovf |= wp::warp_bal<MC, true, 1>(U, 1, W, ureg);
        int32_t* ub = ubuf + (size_t)m * L.ustride;
#pragma unroll
        for (int j = 0; j < MC; j++) {
          const int d = lane * MC + j - 2;
          if (d >= 0 && d < W) ub[d] = ureg[0][j];
        }
      }
      __syncthreads();  // [A2] U digits

      // ---- phase 2b: U^m (x) C_i in chunks of 32 digits of U, one warp per (variable, chunk):
      // operands in registers, fully unrolled (a lone warp pays ~5 cycles per instruction, so the
      // product is spread over the warps that would otherwise wait)
      for (int job = warp; job < D * L.nch; job += kWarps) {
        const int jm = job / L.nch, ch = job - jm * L.nch;
        const int p0 = ch * kPC;
        const int4* up = (const int4*)(ubuf + (size_t)jm * L.ustride + p0);
        int32_t a[kPC];
#pragma unroll
        for (int t4 = 0; t4 < kPC / 4; t4++) {
          const int4 v4 = up[t4];
          a[4 * t4] = v4.x;
          a[4 * t4 + 1] = v4.y;
          a[4 * t4 + 2] = v4.z;
          a[4 * t4 + 3] = v4.w;
        }
        // x[j] = sum_t a[t] C[c_j + Tc - p0 - t], c_j = MC lane + j: a (kPC + MC - 1)-digit window of C_i
        const int32_t* cp = bbuf + lane * MC + Tc - p0 - (kPC - 1);
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
        for (int j = 0; j < MC; j++) xpart[(size_t)job * kCols + lane * MC + j] = okc[j] ? x[j] : 0;
        if (mc) {
          mc->executed += (unsigned long long)kPC;
          mc->useful += (unsigned long long)kPC / 2 + 1;
        }
      }
      __syncthreads();  // [A3] chunk vectors

      // ---- phase 2c: warp m rounds the new row
      if (target) {
        int64_t x[1][MC];
#pragma unroll
        for (int j = 0; j < MC; j++) x[0][j] = 0;
        for (int ch = 0; ch < L.nch; ch++) {
#pragma unroll
          for (int j = 0; j < MC; j++) x[0][j] += xpart[(size_t)(m * L.nch + ch) * kCols + lane * MC + j];
        }
        int32_t rowreg[1][MC];
        ovf |= wp::warp_bal<MC, true, 1>(x, 1, W, rowreg);
        const int z2 = wp::lead_zeros<MC>(rowreg[0], Lf);
#pragma unroll
        for (int j = 0; j < MC; j++) {
          const int d = lane * MC + j - 2;
          if (d >= 0 && d < W) rows[(size_t)(m * N1 + i + 1) * L.stride + d] = rowreg[0][j];
          ssum[j] += rowreg[0][j];
        }
        if (lane == 0) zt[m * N1 + i + 1] = (uint8_t)z2;
      }
      __syncthreads();  // [B] rows i+1 and their zero counts are visible
    }

    if (p.write_coef) {
      int32_t* gcoef = p.coef + (size_t)traj * D * N1 * p.RS;
      // rows leave the kernel in canonical form: sd of the value the semi-normal digits hold
#pragma unroll 1
      for (int r = warp; r < D * N1; r += kWarps) {
        int64_t cv[1][MC];
        int32_t ce[1][MC];
#pragma unroll
        for (int j = 0; j < MC; j++) {
          const int d = lane * MC + j - 2;
          cv[0][j] = (d >= 0 && d < W) ? rows[(size_t)r * L.stride + d] : 0;
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
        if (d >= 0 && d < L.sw) scr[m * L.sw + d] = d < W ? ssum[j] : 0;
      }
      __syncwarp();
      ovf |= warp_normalize_small(scr + (size_t)m * L.sw, L.sw, 0, W, st + (size_t)m * p.RS, &stinfo[m], p.P);
      __syncwarp();
      if ((n % p.stride == 0) || (n == p.n_steps)) {
        const int slot = (n % p.stride == 0) ? (n / p.stride - p.start_step / p.stride)
                                             : (p.n_steps / p.stride - p.start_step / p.stride + 1);
        int32_t* dst = p.rec + ((size_t)slot * p.n_traj + traj) * D * p.RS + (size_t)m * p.RS;
        for (int d = lane; d < p.RS; d += 32) dst[d] = d < W ? st[m * p.RS + d] : 0;
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < D * p.RS; e += kThreads) gstate[e] = (e % p.RS) < W ? st[e] : 0;
  if (ovf && lane == 0) atomicOr(&s_ovf, 1);
  __syncthreads();
  if (tid == 0) p.status[traj] = s_ovf ? kOverflow : kOk;
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
}

}  // namespace blk

bool block_supported(const Params& p) {
  const int passes = (p.N + 32 * blk::kPairWarps) / (32 * blk::kPairWarps);
  return p.D <= blk::DT && p.all_q_small && p.NP >= 1 && p.NP <= 2 && p.Lf + 3 <= blk::kMaxNU && p.Lf >= 3 &&
         passes * (p.Lf + 3) <= 500;
}

size_t block_smem_bytes(const Params& p) { return blk::make_layout(p).total; }

cudaError_t launch_block_kernel(const Params& p, cudaStream_t stream) {
  const void* fn = (const void*)blk::taylor_block_kernel;
  const size_t smem = block_smem_bytes(p);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  Params pp = p;
  void* args[] = {(void*)&pp};
  return cudaLaunchKernel(fn, dim3(p.n_traj), dim3(blk::kThreads), args, smem, stream);
}

}  // namespace mpt
