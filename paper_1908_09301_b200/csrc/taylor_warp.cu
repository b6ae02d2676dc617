// Warp kernel ("warp"): one trajectory per WARP, coefficient rows resident in
// shared memory, no CTA barriers -- ensembles at small precision (W <= 34
// digits: configs[4] at K = 100, 200 and their verify runs) and small single
// trajectories (configs[0]).
//
// Arithmetic (restated bit for bit by oracle/fixmodel.c jet_wp, variant 3): the
// per-order recurrence of the reference's taylor.py:117 _jet_rows, tau-scaled,
//
//   a~_0^m     = sd(state^m)
//   U_i^m      = rndb( [i==0] cst_m B^2 + sum_j tprod(lin[m][j], a~_i^j)
//                      + sum_{t in m} q_t sum_{k<=i} tprod(a~^a_{i-k}, a~^b_k) )      (reduction.py:149 convolve)
//   a~_{i+1}^m = rndb( tprod(U_i^m, C_i) ),     state' = RN_P(sum_i a~_i)            (taylor.py:168 horner_eval)
//
// where every rounding is a function of the VALUE of an exact column sum (sd
// recoding of the two's-complement digits), so zero-digit skipping, folds and
// the order of the partial sums cannot change a bit.
//
// Mapping. Cauchy sums: lane = k. Rows decay with the order, so row j has z_j
// leading zero digits; for order i only the top NU = Lf + 3 - min_k(z_{i-k} +
// z_k) columns of the truncated products are nonzero. Each lane multiplies the
// top-aligned NU-digit windows of its two rows in registers (a fully unrolled
// triangle of NU (NU+1) / 2 IMAD.WIDE, NU rounded up to a multiple of 4 and
// dispatched per order), accumulates its k = lane, lane+32, ... exactly, and
// the 32 lanes reduce-scatter their columns with shuffles. Everything with a
// single product (U x C_i, the non-integer linear term) runs lane = column, the
// left operand broadcast from the lanes that hold its digits. Roundings are
// three parallel carry rounds plus a ballot carry-lookahead (mpt_device.cuh).
#include <cuda_runtime.h>

#include <cstdint>

#include "mpt_common.cuh"
#include "mpt_device.cuh"

namespace mpt {
namespace wp {

constexpr int kLo = 8;      // zero digits stored below digit 0 of every row (window reads reach -5)
constexpr int kMaxNU = 36;  // widest product window => Lf + 3 <= 36
constexpr int kMaxPairs = 4;

struct Layout {
  int ncols, stride, nrows, bw, sw;
  size_t off_rows, off_zt, off_bbuf, off_scr, off_st, total;
};

__host__ __device__ inline Layout make_layout(const Params& p) {
  Layout L;
  L.ncols = p.Lf + 4;                 // relative columns T .. 2 Lf + 1 of every column vector
  L.stride = (kLo + p.W) | 1;         // odd: lanes reading different rows hit different banks
  L.nrows = p.D * (p.N + 1);
  L.bw = 4 + p.W + p.Lf + 4;          // zero-padded right operand of the lane = column products
  L.sw = p.W + 3;                     // state column sums per variable
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o += (bytes + 15) / 16 * 16;
    return r;
  };
  L.off_rows = take(sizeof(int32_t) * ((size_t)L.nrows * L.stride + 2 * kLo));
  L.off_zt = take((size_t)L.nrows);
  L.off_bbuf = take(sizeof(int32_t) * (size_t)L.bw);
  L.off_scr = take(sizeof(int64_t) * (size_t)p.D * L.sw);
  L.off_st = take(sizeof(int32_t) * (size_t)p.D * p.RS + sizeof(int2) * kMaxD);
  L.total = o;
  return L;
}

__device__ __forceinline__ int64_t madw(int32_t a, int32_t b, int64_t c) {
  int64_t d;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}

// ---------------------------------------------------------------------------
// Digits of R = floor((V + [HALF] B^2/2) / B^2), V = sum_c col[c] B^c, in the
// signed-digit recoding of R's two's-complement digits r_j (oracle sd_cols):
//   e_j = r_j - B t_j + t_{j-1},  t_j = [r_j >= B/2],  e_j in [-B/2, B/2].
// Lane l, slot j holds column l*MC + j on entry and output digit (column - 2)
// on exit (columns 0, 1: 0). Returns the warp-uniform overflow flag (R does
// not fit Wout digits).
template <int MC, bool HALF>
__device__ __forceinline__ bool warp_sd(Blk<MC>& b, int Wout, int32_t (&e)[MC]) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  if (HALF) {
#pragma unroll
    for (int j = 0; j < MC; j++)
      if (lane * MC + j == 1) b.v[j] += kRadix / 2;
  }
  int64_t top = blk_rounds(b, MC);
  top += blk_lookahead(b, MC, 1);
  top += blk_lookahead(b, MC, -1);  // digits in [0, B), signed carry out of the vector in `top`
  uint32_t t[MC];
#pragma unroll
  for (int j = 0; j < MC; j++) t[j] = (lane * MC + j >= 2 && b.v[j] >= kRadix / 2) ? 1u : 0u;
  uint32_t tin = __shfl_up_sync(full, t[MC - 1], 1);
  if (lane == 0) tin = 0;
  const uint32_t tlast = __shfl_sync(full, t[MC - 1], 31);
  bool ovf = (top + (int64_t)tlast) != 0;
#pragma unroll
  for (int j = 0; j < MC; j++) {
    const int c = lane * MC + j;
    const uint32_t tp = j == 0 ? tin : t[j - 1];
    int32_t ev = (int32_t)b.v[j] - (t[j] ? (int32_t)kRadix : 0) + (int32_t)tp;
    if (c < 2) ev = 0;
    e[j] = ev;
    if (c - 2 >= Wout && ev != 0) ovf = true;
  }
  return __any_sync(full, ovf);
}

// leading zero digits of a row held across the lanes (digit d at column d + 2): Lf - top, W for a zero row
template <int MC>
__device__ __forceinline__ int lead_zeros(const int32_t (&e)[MC], int Lf) {
  int tp = -1;
#pragma unroll
  for (int j = 0; j < MC; j++) {
    const unsigned m = __ballot_sync(0xffffffffu, e[j] != 0);
    if (m) tp = max(tp, (31 - __clz(m)) * MC + j - 2);
  }
  return Lf - tp;
}

// ---------------------------------------------------------------------------
// acc[u + v] += a'[u] b'[v] over the triangle u + v < NU; a'[u] = ap[-u], b'[v] = bp[-v]
template <int NU>
__device__ __forceinline__ void tri_mac(int64_t (&acc)[NU], const int32_t* ap, const int32_t* bp) {
  int32_t a[NU], b[NU];
#pragma unroll
  for (int u = 0; u < NU; u++) {
    a[u] = ap[-u];
    b[u] = bp[-u];
  }
#pragma unroll
  for (int u = 0; u < NU; u++)
#pragma unroll
    for (int v = 0; v + u < NU; v++) acc[u + v] = madw(a[u], b[v], acc[u + v]);
}

// Sum over the 32 lanes of their NU columns (acc[r] = column ctop - r), returned
// lane = column: out[j] = column lane*MC + j. Each lane first folds its columns
// once (28 low bits stay, the rest moves one column up), so the cross-lane sums
// stay far from 2^63 whatever the data; the value is unchanged.
template <int NU, int MC>
__device__ __forceinline__ void reduce_cols(int64_t (&acc)[NU], int nureal, int ctop, int64_t (&out)[MC]) {
  constexpr int NP2 = NU <= 4 ? 4 : NU <= 8 ? 8 : NU <= 16 ? 16 : NU <= 32 ? 32 : 64;
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  // columns below the truncation (r >= nureal; at most the last three) are not part of the product
#pragma unroll
  for (int r = (NU >= 3 ? NU - 3 : 0); r < NU; r++)
    if (r >= nureal) acc[r] = 0;
  int64_t v[NP2];
  int64_t x = acc[0] >> kRadixBits;  // leaves the top column: column ctop + 1
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
  // lane l now holds element l / (32 / NP2) (NP2 <= 32) or elements 2l, 2l+1 (NP2 = 64)
#pragma unroll
  for (int j = 0; j < MC; j++) {
    const int c = lane * MC + j;
    const int r = ctop - c;
    int64_t got;
    if (NP2 <= 32) {
      got = __shfl_sync(full, v[0], (r * (32 / (NP2 <= 32 ? NP2 : 32))) & 31);
    } else {
      const int64_t g0 = __shfl_sync(full, v[0], (r >> 1) & 31);
      const int64_t g1 = __shfl_sync(full, v[NP2 > 32 ? 1 : 0], (r >> 1) & 31);
      got = (r & 1) ? g1 : g0;
    }
    out[j] = (r >= 0 && r < nureal) ? got : (r == -1 ? x : 0);
  }
}

struct Ctx {
  const int32_t* rows;  // digit 0 of row 0
  const uint8_t* zt;
  int stride, N1, Lf;
};

// digit products inside the nonzero windows of one lane's product (counters only)
__device__ __forceinline__ unsigned useful_tri(int nureal, int ea, int eb, int wa, int wb) {
  // a' holds real digits for u in [ea, ea + wa), b' for v in [eb, eb + wb); u + v < nureal
  unsigned n = 0;
  for (int u = ea; u < ea + wa && u < nureal; u++) {
    const int vmax = min(eb + wb, nureal - u);
    if (vmax > eb) n += vmax - eb;
  }
  return n;
}

// One Cauchy sum of order i on the warp: sum_k tprod(row(va, i-k), row(vb, k)), columns lane = column
template <int NU, int MC>
__device__ __forceinline__ void cauchy_nu(const Ctx& cx, int va, int vb, int i, int zmin, int64_t (&out)[MC],
                                          MacCount* mc) {
  const int lane = threadIdx.x & 31;
  int64_t acc[NU];
#pragma unroll
  for (int r = 0; r < NU; r++) acc[r] = 0;
  const int nureal = cx.Lf + 3 - zmin;
  for (int k = lane; k <= i; k += 32) {
    const int ra = va * cx.N1 + i - k, rb = vb * cx.N1 + k;
    const int za = cx.zt[ra], zb = cx.zt[rb];
    const int sb = min(zb, zmin), sa = zmin - sb;
    tri_mac<NU>(acc, cx.rows + (size_t)ra * cx.stride + cx.Lf - sa, cx.rows + (size_t)rb * cx.stride + cx.Lf - sb);
    if (mc) {
      mc->useful += useful_tri(nureal, za - sa, zb - sb, cx.Lf + 1 - za, cx.Lf + 1 - zb);
      mc->executed += NU * (NU + 1) / 2;
    }
  }
  __syncwarp();
  reduce_cols<NU, MC>(acc, nureal, cx.Lf + 2 - zmin, out);
}

template <int MC>
__device__ __forceinline__ void cauchy(const Ctx& cx, int va, int vb, int i, int64_t (&out)[MC], MacCount* mc) {
  const int lane = threadIdx.x & 31;
  int z = 255;
  for (int k = lane; k <= i; k += 32) z = min(z, (int)cx.zt[va * cx.N1 + i - k] + (int)cx.zt[vb * cx.N1 + k]);
  const int zmin = __reduce_min_sync(0xffffffffu, z);
  const int nureal = cx.Lf + 3 - zmin;
#pragma unroll
  for (int j = 0; j < MC; j++) out[j] = 0;
  if (nureal <= 0) return;
  switch ((nureal + 3) >> 2) {
    case 1: cauchy_nu<4, MC>(cx, va, vb, i, zmin, out, mc); break;
    case 2: cauchy_nu<8, MC>(cx, va, vb, i, zmin, out, mc); break;
    case 3: cauchy_nu<12, MC>(cx, va, vb, i, zmin, out, mc); break;
    case 4: cauchy_nu<16, MC>(cx, va, vb, i, zmin, out, mc); break;
    case 5: cauchy_nu<20, MC>(cx, va, vb, i, zmin, out, mc); break;
    case 6: cauchy_nu<24, MC>(cx, va, vb, i, zmin, out, mc); break;
    case 7: cauchy_nu<28, MC>(cx, va, vb, i, zmin, out, mc); break;
    case 8: cauchy_nu<32, MC>(cx, va, vb, i, zmin, out, mc); break;
    default:
      if (MC >= 2) cauchy_nu<(MC >= 2 ? kMaxNU : 4), MC>(cx, va, vb, i, zmin, out, mc);
      break;
  }
}

// x[j] (+)= sum_p A[p] B[c + T - p] for column c = lane*MC + j < ncols: A's digit p
// is held by the lane of column p + 2, B sits zero-padded in shared memory
template <int MC>
__device__ __forceinline__ void wide_prod(const int32_t (&areg)[MC], int W, const int32_t* B, int T, int ncols,
                                          int64_t (&x)[MC]) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int32_t* bp[MC];
  bool ok[MC];
#pragma unroll
  for (int j = 0; j < MC; j++) {
    const int c = lane * MC + j;
    ok[j] = c < ncols;
    bp[j] = B + (ok[j] ? c + T : 0);
  }
#pragma unroll 4
  for (int p = 0; p < W; p++) {
    const int col = p + 2;
    int32_t a;
    if (MC == 1) {
      a = __shfl_sync(full, areg[0], col);
    } else {
      const int slot = col % MC;
      int32_t pick = areg[0];
#pragma unroll
      for (int j = 1; j < MC; j++)
        if (slot == j) pick = areg[j];
      a = __shfl_sync(full, pick, col / MC);
    }
#pragma unroll
    for (int j = 0; j < MC; j++)
      if (ok[j]) x[j] = madw(a, bp[j][-p], x[j]);
  }
}

// ---------------------------------------------------------------------------
template <int MC, int MINB>
__global__ void __launch_bounds__(128, MINB) taylor_warp_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int traj = blockIdx.x * (blockDim.x >> 5) + wib;
  if (traj >= p.n_traj) return;  // whole warps leave; nothing below synchronises the CTA
  const Layout L = make_layout(p);
  unsigned char* base = smem + (size_t)wib * L.total;
  int32_t* rows = (int32_t*)(base + L.off_rows) + kLo;  // digit 0 of row 0
  uint8_t* zt = (uint8_t*)(base + L.off_zt);
  int32_t* bbuf = (int32_t*)(base + L.off_bbuf) + 4;    // B[q], q in [-4, W + Lf + 4)
  int64_t* scr = (int64_t*)(base + L.off_scr);
  int32_t* st = (int32_t*)(base + L.off_st);
  int2* stinfo = (int2*)(st + (size_t)p.D * p.RS);
  const int D = p.D, N = p.N, N1 = p.N + 1, Lf = p.Lf, W = p.W, ncols = L.ncols;
  const int T = Lf - 2, Tc = Lf + p.sc - 2;

  for (size_t w = lane; w < L.total / 4; w += 32) ((int32_t*)base)[w] = 0;
  __syncwarp();
  int32_t* gstate = p.state + (size_t)traj * D * p.RS;
  for (int e = lane; e < D * p.RS; e += 32) st[e] = gstate[e];
  __syncwarp();

  // pm[q][m]: integer multiplier of pair q's Cauchy sum in equation m
  int pm[kMaxPairs][kMaxD];
#pragma unroll
  for (int q = 0; q < kMaxPairs; q++)
#pragma unroll
    for (int m = 0; m < kMaxD; m++) {
      int s = 0;
      for (int t = 0; t < p.NT; t++)
        if (p.tpair[t] == q && p.teq[t] == m) s += p.tq_int[t];
      pm[q][m] = s;
    }

  Ctx cx{rows, zt, L.stride, N1, Lf};
  MacCount mcount;
  MacCount* mc = p.counters ? &mcount : nullptr;
  bool ovf = false;
  int32_t rowreg[kMaxD][MC];   // newest row of every variable: digit (column - 2) per lane slot
  int64_t ssum[kMaxD][MC];     // running sum of the rows (the next state), same layout

  for (int n = p.start_step + 1; n <= p.n_steps; n++) {
    // ---- row 0 = sd(state)
#pragma unroll
    for (int m = 0; m < kMaxD; m++) {
      if (m < D) {
        Blk<MC> b;
#pragma unroll
        for (int j = 0; j < MC; j++) {
          const int d = lane * MC + j - 2;
          b.v[j] = (d >= 0 && d < W) ? st[m * p.RS + d] : 0;
        }
        ovf |= warp_sd<MC, false>(b, W, rowreg[m]);
        const int z = lead_zeros<MC>(rowreg[m], Lf);
#pragma unroll
        for (int j = 0; j < MC; j++) {
          const int d = lane * MC + j - 2;
          if (d >= 0 && d < W) rows[(size_t)(m * N1) * L.stride + d] = rowreg[m][j];
          ssum[m][j] = rowreg[m][j];
        }
        if (lane == 0) zt[m * N1] = (uint8_t)z;
      }
    }
    __syncwarp();

    for (int i = 0; i < N; i++) {
      int64_t U[kMaxD][MC];
      // ---- constant and linear terms
#pragma unroll
      for (int m = 0; m < kMaxD; m++) {
#pragma unroll
        for (int j = 0; j < MC; j++) U[m][j] = 0;
        if (m < D) {
          if (i == 0) {
#pragma unroll
            for (int j = 0; j < MC; j++) {
              const int d = lane * MC + j - 2;
              if (d >= 0 && d < W) U[m][j] = __ldg(p.cst + (size_t)m * p.RS + d);
            }
          }
#pragma unroll
          for (int jv = 0; jv < kMaxD; jv++) {
            if (jv < D) {
              const int e = m * D + jv;
              if (p.lin_small[e]) {
                const int kq = p.lin_int[e];
                if (kq != 0) {
#pragma unroll
                  for (int j = 0; j < MC; j++) U[m][j] += (int64_t)kq * rowreg[jv][j];
                }
              } else {
                __syncwarp();
                for (int d = lane; d < W; d += 32) bbuf[d] = __ldg(p.lin + (size_t)e * p.RS + d);
                __syncwarp();
                wide_prod<MC>(rowreg[jv], W, bbuf, T, ncols, U[m]);
                if (mc) mc->executed += (unsigned long long)W, mc->useful += (unsigned long long)(W - zt[jv * N1 + i]) / 2 + 1;
              }
            }
          }
        }
      }
      // ---- Cauchy sums
#pragma unroll
      for (int q = 0; q < kMaxPairs; q++) {
        if (q < p.NP) {
          int64_t colv[MC];
          cauchy<MC>(cx, p.pj[q], p.pk[q], i, colv, mc);
#pragma unroll
          for (int m = 0; m < kMaxD; m++)
            if (pm[q][m] != 0) {
#pragma unroll
              for (int j = 0; j < MC; j++) U[m][j] += (int64_t)pm[q][m] * colv[j];
            }
        }
      }
      // ---- U_i = rndb(...), then a~_{i+1} = rndb(U_i (x) C_i)
      int32_t ureg[kMaxD][MC];
#pragma unroll
      for (int m = 0; m < kMaxD; m++) {
        if (m < D) {
          Blk<MC> b;
#pragma unroll
          for (int j = 0; j < MC; j++) b.v[j] = U[m][j];
          ovf |= warp_sd<MC, true>(b, W, ureg[m]);
        }
      }
      __syncwarp();
      for (int d = lane; d < W; d += 32) bbuf[d] = __ldg(p.ctab + (size_t)i * p.RS + d);
      __syncwarp();
#pragma unroll
      for (int m = 0; m < kMaxD; m++) {
        if (m < D) {
          int64_t x[MC];
#pragma unroll
          for (int j = 0; j < MC; j++) x[j] = 0;
          wide_prod<MC>(ureg[m], W, bbuf, Tc, ncols, x);
          Blk<MC> b;
#pragma unroll
          for (int j = 0; j < MC; j++) b.v[j] = x[j];
          ovf |= warp_sd<MC, true>(b, W, rowreg[m]);
          const int z = lead_zeros<MC>(rowreg[m], Lf);
#pragma unroll
          for (int j = 0; j < MC; j++) {
            const int d = lane * MC + j - 2;
            if (d >= 0 && d < W) rows[(size_t)(m * N1 + i + 1) * L.stride + d] = rowreg[m][j];
            ssum[m][j] += rowreg[m][j];
          }
          if (lane == 0) zt[m * N1 + i + 1] = (uint8_t)z;
          if (mc) mc->executed += (unsigned long long)W, mc->useful += (unsigned long long)W / 2 + 1;
        }
      }
      __syncwarp();
    }

    // ---- the jet, when asked for (compute_jet)
    if (p.write_coef) {
      int32_t* gcoef = p.coef + (size_t)traj * D * N1 * p.RS;
      for (int r = 0; r < D * N1; r++)
        for (int d = lane; d < p.RS; d += 32) gcoef[(size_t)r * p.RS + d] = d < W ? rows[(size_t)r * L.stride + d] : 0;
    }
    // ---- state = RN_P(sum of the rows)
#pragma unroll
    for (int m = 0; m < kMaxD; m++) {
      if (m < D) {
#pragma unroll
        for (int j = 0; j < MC; j++) {
          const int d = lane * MC + j - 2;
          if (d >= 0 && d < L.sw) scr[m * L.sw + d] = d < W ? ssum[m][j] : 0;
        }
      }
    }
    __syncwarp();
#pragma unroll 1
    for (int m = 0; m < D; m++) {
      ovf |= warp_normalize_small(scr + (size_t)m * L.sw, L.sw, 0, W, st + (size_t)m * p.RS, &stinfo[m], p.P);
      __syncwarp();
    }
    if ((n % p.stride == 0) || (n == p.n_steps)) {
      const int slot = (n % p.stride == 0) ? (n / p.stride - p.start_step / p.stride)
                                           : (p.n_steps / p.stride - p.start_step / p.stride + 1);
      int32_t* dst = p.rec + ((size_t)slot * p.n_traj + traj) * D * p.RS;
      for (int e = lane; e < D * p.RS; e += 32) dst[e] = (e % p.RS) < W ? st[e] : 0;
    }
    __syncwarp();
  }
  for (int e = lane; e < D * p.RS; e += 32) gstate[e] = (e % p.RS) < W ? st[e] : 0;
  if (lane == 0) p.status[traj] = ovf ? kOverflow : kOk;
  if (mc) {
    unsigned long long u = mcount.useful, x = mcount.executed;
    for (int s = 16; s >= 1; s >>= 1) {
      u += __shfl_xor_sync(full, u, s);
      x += __shfl_xor_sync(full, x, s);
    }
    if (lane == 0) {
      atomicAdd(p.counters, u);
      atomicAdd(p.counters + 1, x);
    }
  }
}

}  // namespace wp

// ---------------------------------------------------------------------------
bool warp_supported(const Params& p) {
  const int passes = (p.N + 1 + 31) / 32;
  // one lane accumulates passes x NU products of at most 2^54 each in int64
  return p.D <= kMaxD && p.all_q_small && p.NP <= wp::kMaxPairs && p.Lf + 3 <= wp::kMaxNU && p.Lf >= 3 &&
         passes * (p.Lf + 3) <= 255 && p.N + 1 < 65536;
}

size_t warp_traj_smem(const Params& p) { return wp::make_layout(p).total; }

static const void* warp_fn(const Params& p) {
  const bool two = p.Lf + 4 > 32;
  return two ? (const void*)wp::taylor_warp_kernel<2, 1> : (const void*)wp::taylor_warp_kernel<1, 3>;
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
