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
// Mapping. Cauchy sums: the 32 lanes are split into NG groups, one per product
// pair, and a group's lanes take k = l, l + GL, ... Rows decay with the order,
// so row j has z_j leading zero digits; for order i only the top NU = Lf + 3 -
// min_k(z_{i-k} + z_k) columns of the truncated products are nonzero. Each lane
// multiplies the top-aligned NU-digit windows of its two rows in registers (a
// fully unrolled triangle of NU (NU+1) / 2 IMAD.WIDE, NU rounded up to a
// multiple of 4 and dispatched per order), accumulates its k's exactly, and the
// lanes of a group reduce-scatter their columns with shuffles -- one butterfly
// per order for all pairs. Everything with a single product (U x C_i, the
// non-integer linear term) runs lane = column with the left operand broadcast
// from shared memory; the D products U^m x C_i share every load of C_i.
// Roundings: all columns are biased positive (a representation of zero is
// added), three parallel carry rounds (the last two in 32 bits), one ballot
// carry-lookahead, then the local sd recoding; the D vectors of a stage are
// processed together so their shuffle latencies overlap.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "mpt_common.cuh"
#include "mpt_device.cuh"

namespace mpt {
namespace wp {

constexpr int kLo = 6;      // zero digits stored below digit 0 of every row (window reads reach -5)
constexpr int kMaxNU = 36;  // widest product window => Lf + 3 <= 36
constexpr int kMaxPairs = 4;

struct Layout {
  int ncols, stride, nrows, bw, sw, nbig;
  size_t off_rows, off_zt, off_bbuf, off_lbuf, off_ubuf, off_scr, off_st, total;
};

__host__ __device__ inline int n_big_lin(const Params& p) {
  int n = 0;
  for (int e = 0; e < p.D * p.D; e++) n += p.lin_small[e] ? 0 : 1;
  return n;
}

__host__ __device__ inline Layout make_layout(const Params& p) {
  Layout L;
  L.ncols = p.Lf + 4;                 // relative columns T .. 2 Lf + 1 of every column vector
  L.stride = (kLo + p.W) | 1;         // odd: lanes reading different rows hit different banks
  L.nrows = p.D * (p.N + 1);
  L.bw = 4 + p.W + p.Lf + 4;          // zero-padded right operand of the lane = column products
  L.sw = p.W + 3;                     // state column sums per variable
  L.nbig = n_big_lin(p);
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
  L.off_ubuf = take(sizeof(int32_t) * 4 * (size_t)p.W);
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
// Digits of R = floor((V + [HALF] B^2/2) / B^2), V = sum_c col[c] B^c, |col[c]| <
// 2^61, in the signed-digit recoding of R's two's-complement digits r_j (oracle
// sd_cols):  e_j = r_j - B t_j + t_{j-1},  t_j = [r_j >= B/2],  e_j in [-B/2, B/2].
// NV vectors at once; lane l, slot j holds column l*MC + j on entry and output
// digit (column - 2) on exit (columns 0, 1: 0). Returns the warp-uniform
// overflow flag (some R does not fit Wout digits).
template <int MC, bool HALF, int NV>
__device__ __forceinline__ bool warp_sd(int64_t (&v)[NV][MC], int nv, int Wout, int32_t (&e)[NV][MC]) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  constexpr int64_t O = int64_t(1) << 62, OB = int64_t(1) << (62 - kRadixBits);
  // bias: a representation of zero that makes every column but the top one positive
  bool istop[MC];
  int64_t bias[MC];
#pragma unroll
  for (int j = 0; j < MC; j++) {
    const int c = lane * MC + j;
    istop[j] = c == 32 * MC - 1;
    bias[j] = istop[j] ? -OB : (c == 0 ? O : O - OB);
    if (HALF && c == 1) bias[j] += kRadix / 2;
  }
  int64_t tval[NV];   // the top column (lane 31, last slot) absorbs; signed
  uint32_t w[NV][MC];
  {
    // round 1 (64 bits)
    uint32_t d1[NV][MC];
    uint64_t k1[NV][MC];
#pragma unroll
    for (int m = 0; m < NV; m++) {
      tval[m] = 0;
#pragma unroll
      for (int j = 0; j < MC; j++) {
        const int64_t s = v[m][j] + bias[j];
        if (istop[j]) tval[m] = s;
        d1[m][j] = istop[j] ? 0u : ((uint32_t)s & (uint32_t)kMask);
        k1[m][j] = istop[j] ? 0ull : ((uint64_t)s >> kRadixBits);
      }
    }
    uint64_t kin[NV];
#pragma unroll
    for (int m = 0; m < NV; m++) kin[m] = __shfl_up_sync(full, k1[m][MC - 1], 1);
    // round 2 (carries < 2^36 in, < 2^8 out)
    uint32_t d2[NV][MC], k2[NV][MC];
#pragma unroll
    for (int m = 0; m < NV; m++) {
#pragma unroll
      for (int j = 0; j < MC; j++) {
        const uint64_t cin = j == 0 ? (lane == 0 ? 0ull : kin[m]) : k1[m][j - 1];
        const uint64_t w1 = (uint64_t)d1[m][j] + cin;
        if (istop[j]) tval[m] += (int64_t)cin;
        d2[m][j] = istop[j] ? 0u : ((uint32_t)w1 & (uint32_t)kMask);
        k2[m][j] = istop[j] ? 0u : (uint32_t)(w1 >> kRadixBits);
      }
    }
    uint32_t kin2[NV];
#pragma unroll
    for (int m = 0; m < NV; m++) kin2[m] = __shfl_up_sync(full, k2[m][MC - 1], 1);
    // round 3 (32 bits): carries in {0, 1} out
    uint32_t d3[NV][MC], k3[NV][MC];
#pragma unroll
    for (int m = 0; m < NV; m++) {
#pragma unroll
      for (int j = 0; j < MC; j++) {
        const uint32_t cin = j == 0 ? (lane == 0 ? 0u : kin2[m]) : k2[m][j - 1];
        const uint32_t w2 = d2[m][j] + cin;
        if (istop[j]) tval[m] += cin;
        d3[m][j] = istop[j] ? 0u : (w2 & (uint32_t)kMask);
        k3[m][j] = istop[j] ? 0u : (w2 >> kRadixBits);
      }
    }
    uint32_t kin3[NV];
#pragma unroll
    for (int m = 0; m < NV; m++) kin3[m] = __shfl_up_sync(full, k3[m][MC - 1], 1);
#pragma unroll
    for (int m = 0; m < NV; m++) {
#pragma unroll
      for (int j = 0; j < MC; j++) {
        const uint32_t cin = j == 0 ? (lane == 0 ? 0u : kin3[m]) : k3[m][j - 1];
        if (istop[j]) tval[m] += cin;
        w[m][j] = d3[m][j] + cin;  // in [0, B]
      }
    }
  }
  // carry lookahead for the remaining +1 ripples: a column generates when it equals B,
  // propagates when it equals B - 1 (the top column does neither)
  uint32_t gl[NV], pl[NV];
#pragma unroll
  for (int m = 0; m < NV; m++) {
    bool g = false, pr = true;
#pragma unroll
    for (int j = 0; j < MC; j++) {
      const bool gj = !istop[j] && (w[m][j] >> kRadixBits) != 0;
      const bool pj = !istop[j] && w[m][j] == (uint32_t)kMask;
      g = gj || (pj && g);  // lane-level generate / propagate over its MC columns
      pr = pr && pj;
    }
    gl[m] = __ballot_sync(full, g);
    pl[m] = __ballot_sync(full, pr);
  }
  bool ovf = false;
#pragma unroll
  for (int m = 0; m < NV; m++) {
    const uint32_t cmask = ((gl[m] | pl[m]) + gl[m]) ^ pl[m];  // bit l: carry into lane l
    uint32_t cin = (cmask >> lane) & 1u;
    uint32_t r[MC];
#pragma unroll
    for (int j = 0; j < MC; j++) {
      const uint32_t s = w[m][j] + cin;
      if (istop[j]) {
        tval[m] += cin;
        r[j] = (uint32_t)tval[m] & (uint32_t)kMask;
      } else {
        r[j] = s & (uint32_t)kMask;
        cin = s >> kRadixBits;
      }
    }
    // sd recoding
    uint32_t t[MC];
#pragma unroll
    for (int j = 0; j < MC; j++) t[j] = (lane * MC + j >= 2 && r[j] >= (uint32_t)(kRadix / 2)) ? 1u : 0u;
    uint32_t tin = __shfl_up_sync(full, t[MC - 1], 1);
    if (lane == 0) tin = 0;
#pragma unroll
    for (int j = 0; j < MC; j++) {
      const int c = lane * MC + j;
      const uint32_t tp = j == 0 ? tin : t[j - 1];
      int32_t ev = (int32_t)r[j] - (t[j] ? (int32_t)kRadix : 0) + (int32_t)tp;
      if (c < 2) ev = 0;
      e[m][j] = ev;
      if (m < nv && c - 2 >= Wout && ev != 0) ovf = true;
    }
    if (m < nv && lane == 31 && ((tval[m] >> kRadixBits) + (int64_t)t[MC - 1]) != 0) ovf = true;
  }
  return __any_sync(full, ovf);
}

// ---------------------------------------------------------------------------
// The same value R = floor((V + [HALF] B^2/2) / B^2) in BALANCED SEMI-NORMAL digits:
// e_j in [-B/2 - 1, B/2], sum_j e_j B^j = R exactly, three parallel carry rounds
// and nothing else (no carry lookahead, no recoding). Every consumer of U and
// of the coefficient rows is an exact integer product or sum, so only the VALUE
// matters; the canonical digits (warp_sd of the same value) are produced when a
// row leaves the kernel (compute_jet). Columns 0 and 1 are split by floor, so
// after two rounds nothing more can leave them: the truncation is exact.
template <int MC, bool HALF, int NV>
__device__ __forceinline__ bool warp_bal(int64_t (&v)[NV][MC], int nv, int Wout, int32_t (&e)[NV][MC]) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  constexpr int32_t HB = (int32_t)(kRadix / 2);
  bool istop[MC];
  int32_t off[MC];
#pragma unroll
  for (int j = 0; j < MC; j++) {
    const int c = lane * MC + j;
    istop[j] = c == 32 * MC - 1;
    off[j] = c < 2 ? 0 : HB;
  }
  int64_t tval[NV];
  int32_t d1[NV][MC];
  int64_t k1[NV][MC];
#pragma unroll
  for (int m = 0; m < NV; m++) {
    tval[m] = 0;
#pragma unroll
    for (int j = 0; j < MC; j++) {
      int64_t t = v[m][j] + off[j];
      if (HALF && lane * MC + j == 1) t += HB;
      if (istop[j]) tval[m] = v[m][j];
      d1[m][j] = istop[j] ? 0 : (int32_t)((uint32_t)t & (uint32_t)kMask) - off[j];
      k1[m][j] = istop[j] ? 0 : (t >> kRadixBits);
    }
  }
  int64_t kin[NV];
#pragma unroll
  for (int m = 0; m < NV; m++) kin[m] = __shfl_up_sync(full, k1[m][MC - 1], 1);
  // round 2 (carries < 2^35 in, < 2^8 out)
  int32_t d2[NV][MC], k2[NV][MC];
#pragma unroll
  for (int m = 0; m < NV; m++) {
#pragma unroll
    for (int j = 0; j < MC; j++) {
      const int64_t cin = j == 0 ? (lane == 0 ? 0ll : kin[m]) : k1[m][j - 1];
      if (istop[j]) tval[m] += cin;
      const int64_t t = (int64_t)d1[m][j] + cin + off[j];
      d2[m][j] = istop[j] ? 0 : (int32_t)((uint32_t)t & (uint32_t)kMask) - off[j];
      k2[m][j] = istop[j] ? 0 : (int32_t)(t >> kRadixBits);
    }
  }
  int32_t kin2[NV];
#pragma unroll
  for (int m = 0; m < NV; m++) kin2[m] = __shfl_up_sync(full, k2[m][MC - 1], 1);
  // round 3 (32 bits): carries in {-1, 0, 1} out
  int32_t d3[NV][MC], k3[NV][MC];
#pragma unroll
  for (int m = 0; m < NV; m++) {
#pragma unroll
    for (int j = 0; j < MC; j++) {
      const int32_t cin = j == 0 ? (lane == 0 ? 0 : kin2[m]) : k2[m][j - 1];
      if (istop[j]) tval[m] += cin;
      const int32_t t = d2[m][j] + cin + off[j];
      d3[m][j] = istop[j] ? 0 : (int32_t)((uint32_t)t & (uint32_t)kMask) - off[j];
      k3[m][j] = istop[j] ? 0 : (t >> kRadixBits);
    }
  }
  int32_t kin3[NV];
#pragma unroll
  for (int m = 0; m < NV; m++) kin3[m] = __shfl_up_sync(full, k3[m][MC - 1], 1);
  bool ovf = false;
#pragma unroll
  for (int m = 0; m < NV; m++) {
#pragma unroll
    for (int j = 0; j < MC; j++) {
      const int c = lane * MC + j;
      const int32_t cin = j == 0 ? (lane == 0 ? 0 : kin3[m]) : k3[m][j - 1];
      int32_t ev;
      if (istop[j]) {
        tval[m] += cin;
        ev = (int32_t)tval[m];
        if (m < nv && (tval[m] > HB || tval[m] < -HB)) ovf = true;
      } else {
        ev = d3[m][j] + cin;
      }
      if (c < 2) ev = 0;
      e[m][j] = ev;
      if (m < nv && c - 2 >= Wout && ev != 0) ovf = true;
    }
  }
  return __any_sync(full, ovf);
}

// the rounding the kernels use inside their loops (MPT_CANONICAL_ROUNDING: the canonical
// digits everywhere, for A/B timing of the semi-normal representation)
template <int MC, bool HALF, int NV>
__device__ __forceinline__ bool warp_rnd(int64_t (&v)[NV][MC], int nv, int Wout, int32_t (&e)[NV][MC]) {
#ifdef MPT_CANONICAL_ROUNDING
  return warp_sd<MC, HALF, NV>(v, nv, Wout, e);
#else
  return warp_bal<MC, HALF, NV>(v, nv, Wout, e);
#endif
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

struct Ctx {
  const int32_t* rows;  // digit 0 of row 0
  const uint8_t* zt;
  int stride, N1, Lf, NP;
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

// The Cauchy sums of order i of every pair at once: group g = lane / GL works on
// pair g, its lanes on k = l, l + GL, ...; acc[r] = column ctop - r. After the
// products each lane folds its columns once (28 low bits stay, the rest moves one
// column up: the cross-lane sums stay far from 2^63 whatever the data), the GL
// lanes of a group reduce-scatter them with shuffles, and every lane fetches
// column lane*MC + j of pair q into out[q][j].
template <int NU, int MC, int NG>
__device__ __forceinline__ void cauchy_nu(const Ctx& cx, int va, int vb, int i, int zmin, int64_t (&out)[NG][MC],
                                          MacCount* mc) {
  constexpr int GL = 32 / NG;
  constexpr int NP2 = NU <= 4 ? 4 : NU <= 8 ? 8 : NU <= 16 ? 16 : NU <= 32 ? 32 : 64;
  constexpr int E = NP2 >= GL ? NP2 / GL : 1;  // elements a lane ends up with
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31, grp = lane / GL, l = lane % GL;
  const int nureal = cx.Lf + 3 - zmin, ctop = cx.Lf + 2 - zmin;
  int64_t acc[NU];
#pragma unroll
  for (int r = 0; r < NU; r++) acc[r] = 0;
  if (grp < cx.NP) {
    for (int k = l; k <= i; k += GL) {
      const int ra = va * cx.N1 + i - k, rb = vb * cx.N1 + k;
      const int za = cx.zt[ra], zb = cx.zt[rb];
      const int sb = min(zb, zmin), sa = zmin - sb;
      tri_mac<NU>(acc, cx.rows + (size_t)ra * cx.stride + cx.Lf - sa, cx.rows + (size_t)rb * cx.stride + cx.Lf - sb);
      if (mc) {
        mc->useful += useful_tri(nureal, za - sa, zb - sb, cx.Lf + 1 - za, cx.Lf + 1 - zb);
        mc->executed += NU * (NU + 1) / 2;
      }
    }
  }
  __syncwarp();
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
  for (int s = GL / 2; s >= 1; s >>= 1) {
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
  // group lane l now holds elements [l E, l E + E) (NP2 >= GL) or element l / (GL / NP2)
#pragma unroll
  for (int q = 0; q < NG; q++) {
#pragma unroll
    for (int j = 0; j < MC; j++) {
      const int c = lane * MC + j;
      const int r = ctop - c;
      const int holder = NP2 >= GL ? r / E : r * (GL / (NP2 >= GL ? GL : NP2));
      const int src = (q * GL + (holder & (GL - 1))) & 31;
      int64_t got = 0;
#pragma unroll
      for (int ee = 0; ee < E; ee++) {
        const int64_t g = __shfl_sync(full, v[ee], src);
        if ((r & (E - 1)) == ee) got = g;
      }
      const int64_t xq = __shfl_sync(full, x, q * GL);
      out[q][j] = (r >= 0 && r < nureal) ? got : (r == -1 ? xq : 0);
    }
  }
}

template <int MC, int NG>
__device__ __forceinline__ void cauchy(const Ctx& cx, int va, int vb, int i, int64_t (&out)[NG][MC], MacCount* mc) {
  constexpr int GL = 32 / NG;
  const int lane = threadIdx.x & 31, grp = lane / GL, l = lane % GL;
  int z = 255;
  if (grp < cx.NP)
    for (int k = l; k <= i; k += GL) z = min(z, (int)cx.zt[va * cx.N1 + i - k] + (int)cx.zt[vb * cx.N1 + k]);
  const int zmin = __reduce_min_sync(0xffffffffu, z);
  const int nureal = cx.Lf + 3 - zmin;
  if (nureal <= 0) {
#pragma unroll
    for (int q = 0; q < NG; q++)
#pragma unroll
      for (int j = 0; j < MC; j++) out[q][j] = 0;
    return;
  }
  switch ((nureal + 3) >> 2) {
    case 1: cauchy_nu<4, MC, NG>(cx, va, vb, i, zmin, out, mc); break;
    case 2: cauchy_nu<8, MC, NG>(cx, va, vb, i, zmin, out, mc); break;
    case 3: cauchy_nu<12, MC, NG>(cx, va, vb, i, zmin, out, mc); break;
    case 4: cauchy_nu<16, MC, NG>(cx, va, vb, i, zmin, out, mc); break;
    case 5: cauchy_nu<20, MC, NG>(cx, va, vb, i, zmin, out, mc); break;
    case 6: cauchy_nu<24, MC, NG>(cx, va, vb, i, zmin, out, mc); break;
    case 7: cauchy_nu<28, MC, NG>(cx, va, vb, i, zmin, out, mc); break;
    case 8: cauchy_nu<32, MC, NG>(cx, va, vb, i, zmin, out, mc); break;
    default: cauchy_nu<(MC >= 2 ? kMaxNU : 32), MC, NG>(cx, va, vb, i, zmin, out, mc); break;
  }
}

// ---------------------------------------------------------------------------
// MC columns per lane, DT >= D variables unrolled, NG lane groups (>= pairs)
template <int MC, int DT, int NG, int MINB>
__global__ void __launch_bounds__(128, MINB) taylor_warp_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const unsigned full = 0xffffffffu;
  constexpr int GL = 32 / NG;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int traj = blockIdx.x * (blockDim.x >> 5) + wib;
  if (traj >= p.n_traj) return;  // whole warps leave; nothing below synchronises the CTA
  const Layout L = make_layout(p);
  unsigned char* base = smem + (size_t)wib * L.total;
  int32_t* rows = (int32_t*)(base + L.off_rows) + kLo;  // digit 0 of row 0
  uint8_t* zt = (uint8_t*)(base + L.off_zt);
  int32_t* bbuf = (int32_t*)(base + L.off_bbuf) + 4;    // B[q], q in [-4, W + Lf + 4)
  int32_t* lbuf = (int32_t*)(base + L.off_lbuf) + 4;    // the non-integer linear coefficients, same padding
  int32_t* ubuf = (int32_t*)(base + L.off_ubuf);        // U digits, [p][4]
  int64_t* scr = (int64_t*)(base + L.off_scr);
  int32_t* st = (int32_t*)(base + L.off_st);
  int2* stinfo = (int2*)(st + (size_t)p.D * p.RS);
  const int D = p.D, N = p.N, N1 = p.N + 1, Lf = p.Lf, W = p.W, ncols = L.ncols;
  const int T = Lf - 2, Tc = Lf + p.sc - 2;

  for (size_t w = lane; w < L.total / 4; w += 32) ((int32_t*)base)[w] = 0;
  __syncwarp();
  int32_t* gstate = p.state + (size_t)traj * D * p.RS;
  for (int e = lane; e < D * p.RS; e += 32) st[e] = gstate[e];
  {
    int slot = 0;
    for (int e = 0; e < D * D; e++) {
      if (p.lin_small[e]) continue;
      for (int d = lane; d < W; d += 32) lbuf[(size_t)slot * L.bw + d] = p.lin[(size_t)e * p.RS + d];
      slot++;
    }
  }
  __syncwarp();

  // this lane's pair (group), column flags, constant term
  const int grp = lane / GL;
  const int va = grp < p.NP ? p.pj[grp] : 0, vb = grp < p.NP ? p.pk[grp] : 0;
  bool okc[MC];
  int32_t cstreg[DT][MC];
#pragma unroll
  for (int j = 0; j < MC; j++) {
    const int c = lane * MC + j;
    okc[j] = c < ncols;
#pragma unroll
    for (int m = 0; m < DT; m++) {
      const int d = c - 2;
      cstreg[m][j] = (m < D && d >= 0 && d < W) ? p.cst[(size_t)m * p.RS + d] : 0;
    }
  }

  // per-kernel tables in registers: integer multiplier of pair q in equation m, integer
  // linear coefficients, and which linear entries need a full product (bit m*DT + jv)
  int pm[NG][DT], linint[DT][DT];
  unsigned bigmask = 0;
#pragma unroll
  for (int m = 0; m < DT; m++) {
#pragma unroll
    for (int q = 0; q < NG; q++) {
      int s = 0;
      for (int t = 0; t < p.NT; t++)
        if (p.tpair[t] == q && p.teq[t] == m) s += p.tq_int[t];
      pm[q][m] = s;
    }
#pragma unroll
    for (int jv = 0; jv < DT; jv++) {
      linint[m][jv] = 0;
      if (m < D && jv < D) {
        if (p.lin_small[m * D + jv])
          linint[m][jv] = p.lin_int[m * D + jv];
        else
          bigmask |= 1u << (m * DT + jv);
      }
    }
  }

  Ctx cx{rows, zt, L.stride, N1, Lf, p.NP};
  MacCount mcount;
  MacCount* mc = p.counters ? &mcount : nullptr;
  bool ovf = false;
  int32_t rowreg[DT][MC];   // newest row of every variable: digit (column - 2) per lane slot
  int64_t ssum[DT][MC];     // running sum of the rows (the next state), same layout
  int32_t cnext[2];         // C_i digits lane, lane + 32 (prefetched one order ahead)

  for (int n = p.start_step + 1; n <= p.n_steps; n++) {
    // ---- row 0 = sd(state)
    {
      int64_t v[DT][MC];
#pragma unroll
      for (int m = 0; m < DT; m++)
#pragma unroll
        for (int j = 0; j < MC; j++) {
          const int d = lane * MC + j - 2;
          v[m][j] = (m < D && d >= 0 && d < W) ? st[m * p.RS + d] : 0;
        }
      ovf |= warp_rnd<MC, false, DT>(v, D, W, rowreg);
#pragma unroll
      for (int m = 0; m < DT; m++) {
        if (m < D) {
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
    }
    cnext[0] = lane < W ? __ldg(p.ctab + lane) : 0;
    cnext[1] = lane + 32 < W ? __ldg(p.ctab + lane + 32) : 0;
    __syncwarp();

    for (int i = 0; i < N; i++) {
      int64_t U[DT][MC];
      // ---- C_i into the padded operand buffer, C_{i+1} on its way
      if (lane < W) bbuf[lane] = cnext[0];  // digits >= W of the buffer stay zero
      if (lane + 32 < W) bbuf[lane + 32] = cnext[1];
      if (i + 1 < N) {
        cnext[0] = lane < W ? __ldg(p.ctab + (size_t)(i + 1) * p.RS + lane) : 0;
        cnext[1] = lane + 32 < W ? __ldg(p.ctab + (size_t)(i + 1) * p.RS + lane + 32) : 0;
      }
      // ---- constant and linear terms
#pragma unroll
      for (int m = 0; m < DT; m++) {
#pragma unroll
        for (int j = 0; j < MC; j++) U[m][j] = i == 0 ? (int64_t)cstreg[m][j] : 0;
      }
#pragma unroll
      for (int m = 0; m < DT; m++)
#pragma unroll
        for (int jv = 0; jv < DT; jv++)
          if (linint[m][jv] != 0) {
#pragma unroll
            for (int j = 0; j < MC; j++) U[m][j] += (int64_t)linint[m][jv] * rowreg[jv][j];
          }
      if (bigmask) {
        int slot = 0;
#pragma unroll
        for (int m = 0; m < DT; m++) {
#pragma unroll
          for (int jv = 0; jv < DT; jv++) {
            if (bigmask & (1u << (m * DT + jv))) {
              // tprod(lin[m][jv], a~_i^jv): row digits broadcast from shared memory
              const int32_t* ar = rows + (size_t)(jv * N1 + i) * L.stride;
              const int wa = W - zt[jv * N1 + i];  // digits above are zero
              const int32_t* lb[MC];
#pragma unroll
              for (int j = 0; j < MC; j++) lb[j] = lbuf + (size_t)slot * L.bw + (okc[j] ? lane * MC + j + T : -4);
              // two accumulator chains: the IMAD.WIDE latency, not the pipe, bounds a lone warp
              int64_t y[MC];
#pragma unroll
              for (int j = 0; j < MC; j++) y[j] = 0;
              int pp = 0;
#pragma unroll 2
              for (; pp + 1 < wa; pp += 2) {
                const int32_t a0 = ar[pp], a1 = ar[pp + 1];
#pragma unroll
                for (int j = 0; j < MC; j++) {
                  U[m][j] = madw(a0, lb[j][okc[j] ? -pp : 0], U[m][j]);
                  y[j] = madw(a1, lb[j][okc[j] ? -pp - 1 : 0], y[j]);
                }
              }
              if (pp < wa) {
                const int32_t a0 = ar[pp];
#pragma unroll
                for (int j = 0; j < MC; j++) U[m][j] = madw(a0, lb[j][okc[j] ? -pp : 0], U[m][j]);
              }
#pragma unroll
              for (int j = 0; j < MC; j++) U[m][j] += y[j];
              if (mc) {
                mc->executed += (unsigned long long)wa;
                mc->useful += (unsigned long long)wa / 2 + 1;
              }
              slot++;
            }
          }
        }
      }
      // ---- Cauchy sums of every pair
      if (p.NP > 0) {
        int64_t colv[NG][MC];
        cauchy<MC, NG>(cx, va, vb, i, colv, mc);
#pragma unroll
        for (int q = 0; q < NG; q++) {
          if (q < p.NP) {
#pragma unroll
            for (int m = 0; m < DT; m++) {
              if (pm[q][m] != 0) {
#pragma unroll
                for (int j = 0; j < MC; j++) U[m][j] += (int64_t)pm[q][m] * colv[q][j];
              }
            }
          }
        }
      }
      // ---- U_i = rndb(...), digits to shared memory as [p][m]
      int32_t ureg[DT][MC];
      ovf |= warp_rnd<MC, true, DT>(U, D, W, ureg);
#pragma unroll
      for (int j = 0; j < MC; j++) {
        const int d = lane * MC + j - 2;
        if (d >= 0 && d < W) {
          if (DT == 3)
            *(int4*)(ubuf + 4 * d) = make_int4(ureg[0][j], ureg[1][j], ureg[2][j], 0);
          else
            *(int4*)(ubuf + 4 * d) = make_int4(ureg[0][j], ureg[1][j], ureg[2][j], ureg[DT - 1][j]);
        }
      }
      __syncwarp();
      // ---- a~_{i+1}^m = rndb(U_i^m (x) C_i): the D products share every load of C_i
      int64_t x[DT][MC];
#pragma unroll
      for (int m = 0; m < DT; m++)
#pragma unroll
        for (int j = 0; j < MC; j++) x[m][j] = 0;
      {
        // columns >= ncols read the low zero padding (index -4): no predicates in the loop
        const int32_t* bq[MC];
        int step[MC];
#pragma unroll
        for (int j = 0; j < MC; j++) {
          bq[j] = bbuf + (okc[j] ? lane * MC + j + Tc : -4);
          step[j] = okc[j] ? 1 : 0;
        }
        const int4* up = (const int4*)ubuf;
#pragma unroll 4
        for (int pp = 0; pp < W; pp++) {
          const int4 a4 = up[pp];
#pragma unroll
          for (int j = 0; j < MC; j++) {
            const int32_t b = *bq[j];
            bq[j] -= step[j];
            x[0][j] = madw(a4.x, b, x[0][j]);
            if (DT > 1) x[1][j] = madw(a4.y, b, x[1][j]);
            if (DT > 2) x[2][j] = madw(a4.z, b, x[2][j]);
            if (DT > 3) x[DT - 1][j] = madw(a4.w, b, x[DT - 1][j]);
          }
        }
      }
      if (mc) {
        mc->executed += (unsigned long long)W * D;
        mc->useful += (unsigned long long)(W / 2 + 1) * D;
      }
      ovf |= warp_rnd<MC, true, DT>(x, D, W, rowreg);
#pragma unroll
      for (int m = 0; m < DT; m++) {
        if (m < D) {
          const int z = lead_zeros<MC>(rowreg[m], Lf);
#pragma unroll
          for (int j = 0; j < MC; j++) {
            const int d = lane * MC + j - 2;
            if (d >= 0 && d < W) rows[(size_t)(m * N1 + i + 1) * L.stride + d] = rowreg[m][j];
            ssum[m][j] += rowreg[m][j];
          }
          if (lane == 0) zt[m * N1 + i + 1] = (uint8_t)z;
        }
      }
      __syncwarp();
    }

    // ---- the jet, when asked for (compute_jet)
    if (p.write_coef) {
      // rows leave the kernel in canonical form: sd of the value the semi-normal digits hold
      int32_t* gcoef = p.coef + (size_t)traj * D * N1 * p.RS;
#pragma unroll 1
      for (int r = 0; r < D * N1; r++) {
        int64_t cv[1][MC];
        int32_t ce[1][MC];
#pragma unroll
        for (int j = 0; j < MC; j++) {
          const int d = lane * MC + j - 2;
          cv[0][j] = (d >= 0 && d < W) ? rows[(size_t)r * L.stride + d] : 0;
        }
        warp_sd<MC, false, 1>(cv, 1, W, ce);
#pragma unroll
        for (int j = 0; j < MC; j++) {
          const int d = lane * MC + j - 2;
          if (d >= 0 && d < p.RS) gcoef[(size_t)r * p.RS + d] = d < W ? ce[0][j] : 0;
        }
      }
    }
    // ---- state = RN_P(sum of the rows)
#pragma unroll
    for (int m = 0; m < DT; m++) {
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

// instantiation choice shared by the two translation units (one per MC)
template <int MC>
inline const void* warp_fn_mc(const Params& p) {
  constexpr int MINB = MC == 1 ? 3 : 1;
  if (p.D <= 3 && p.NP <= 2) return (const void*)taylor_warp_kernel<MC, 3, 2, MINB>;
  return (const void*)taylor_warp_kernel<MC, 4, 4, MINB>;
}

}  // namespace wp
}  // namespace mpt
