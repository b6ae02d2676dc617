// Device building blocks shared by the Taylor kernels (sm_100a):
//   * column accumulation of truncated digit products in exact 64-bit integer
//     registers (one IMAD.WIDE per digit product, register window of kR
//     columns, periodic carry folds), with zero-digit skipping;
//   * warp-cooperative carry propagation / rounding of column sums into
//     canonical digits;
//   * rounding of a digit row to the reference precision (ties to even).
// The arithmetic is restated bit for bit by oracle/fixmodel.c.
#pragma once
#include <cstdint>

#include "mpt_common.cuh"

namespace mpt {

// ---------------------------------------------------------------------------
// Column accumulation for one (operand pair, column group).
// acc[r] += sum_p A[p] * B[c0 + r - p] for the group's absolute columns
// c0..c0+kR-1; acc[kR] collects the carries of folds. Rows are padded with
// kPad zeros on both sides so the register window never needs bounds checks.
struct Acc {
  int64_t v[kR + 1];
};

// s64 += s32 * s32 as ONE instruction (SASS IMAD.WIDE); writing the product
// in C++ on int64 operands makes nvcc emit a 64x64 multiply sequence.
__device__ __forceinline__ int64_t mad_wide(int32_t a, int32_t b, int64_t c) {
#ifdef MPT_MAD_ASM
  int64_t d;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
#else
  return c + (int64_t)a * (int64_t)b;
#endif
}

__device__ __forceinline__ void acc_zero(Acc& a) {
#pragma unroll
  for (int r = 0; r <= kR; r++) a.v[r] = 0;
}

// fold: digits of acc[0..kR-1] into [0, B), carries ripple upward into acc[kR].
// Columns below `tcut` (absolute) are discarded first: products there are
// outside the truncated product and must not leak carries upward.
__device__ __forceinline__ void acc_fold(Acc& a, int c0, int tcut) {
#pragma unroll
  for (int r = 0; r < kR; r++) {
    if (c0 + r < tcut) a.v[r] = 0;
    int64_t c = a.v[r] >> kRadixBits;
    a.v[r] &= kMask;
    a.v[r + 1] += c;
  }
}

struct MacCount {
  unsigned long long useful = 0, executed = 0;
};

// exact number of digit products (p, q) inside the nonzero windows that fall
// in the group's kept columns [max(c0, tcut), c0 + kR) -- the algorithmic work
__device__ __forceinline__ unsigned useful_macs(int2 ia, int2 ib, int c0, int tcut) {
  unsigned n = 0;
#pragma unroll
  for (int r = 0; r < kR; r++) {
    int c = c0 + r;
    int lo = max(ia.x, c - ib.y), hi = min(ia.y, c - ib.x);
    if (c >= tcut && hi >= lo) n += hi - lo + 1;
  }
  return n;
}

__device__ __forceinline__ void mac_group(Acc& acc, int& cnt, const int32_t* __restrict__ A, int2 ia,
                                       const int32_t* __restrict__ B, int2 ib, int c0, int tcut,
                                       MacCount* mc = nullptr) {
  // nonzero digits: A in [ia.x, ia.y], B in [ib.x, ib.y]
  int plo = max(ia.x, c0 - ib.y);
  int phi = min(ia.y, c0 + kR - 1 - ib.x);
  if (plo > phi) return;
  int P0 = plo & ~(kR - 1);
  if (mc) {
    mc->useful += useful_macs(ia, ib, c0, tcut);
    mc->executed += (unsigned long long)(((phi - P0) / kR + 1) * kR * kR);
  }
  int32_t buf[kR];
  const int32_t* bq = B + (c0 - P0);  // bq[s] = B[c0 - P0 + s]
#pragma unroll
  for (int s = 1; s < kR; s++) buf[s] = bq[s];
  for (; P0 <= phi; P0 += kR) {
    const int32_t* ap = A + P0;
    const int32_t* bp = B + (c0 - P0);
#pragma unroll
    for (int u = 0; u < kR; u++) {
      buf[(kR - u) & (kR - 1)] = bp[-u];
      const int32_t a = ap[u];
#pragma unroll
      for (int r = 0; r < kR; r++) acc.v[r] = mad_wide(a, buf[(r - u) & (kR - 1)], acc.v[r]);
    }
    cnt += kR;
    if (cnt >= kFoldEvery) {
      acc_fold(acc, c0, tcut);
      cnt = 0;
    }
  }
}

// mac_group restricted to chunk `pc` of `pch` near-equal runs of whole kR
// blocks of the p range: lets several threads share one (row pair, group).
__device__ __forceinline__ void mac_group_chunk(Acc& acc, int& cnt, const int32_t* __restrict__ A, int2 ia,
                                                const int32_t* __restrict__ B, int2 ib, int c0, int tcut, int pc,
                                                int pch, MacCount* mc) {
  if (pch > 1) {
    const int plo = max(ia.x, c0 - ib.y), phi = min(ia.y, c0 + kR - 1 - ib.x);
    if (plo > phi) return;
    const int b0 = plo / kR, nb = phi / kR - b0 + 1;
    const int per = (nb + pch - 1) / pch;
    const int blo = b0 + pc * per, bhi = min(b0 + nb, blo + per) - 1;
    if (blo > bhi) return;
    ia.x = max(ia.x, blo * kR);
    ia.y = min(ia.y, bhi * kR + kR - 1);
  }
  mac_group(acc, cnt, A, ia, B, ib, c0, tcut, mc);
}

// ---------------------------------------------------------------------------
// Warp-cooperative normalisation of a column vector (relative columns
// 0..ncols-1, value V = sum col[c] B^c, |col[c]| < 2^62) into canonical signed
// digits of floor((V + [drop] B^drop / 2) / B^drop), drop in {0, 2}.
// Lane l holds columns [l*m, l*m+m). No data-dependent loops and no long
// per-lane dependency chains:
//   * three rounds of "split every column into digit + carry, add the carry to
//     the next column" (all columns in parallel) leave digits in [-1, B];
//   * one carry-lookahead per sign resolves the remaining +1 / -1 ripples:
//     inside a lane with m-bit generate/propagate masks,
//         C = (((A & P) + P) ^ P) | A,   A = (G << 1) | carry_in,
//     and across lanes with the same identity on __ballot_sync masks.
template <int MM>
struct Blk {
  int64_t v[MM];
};

// three parallel carry rounds; returns what leaves lane 31 (warp-uniform)
template <int MM>
__device__ __forceinline__ int64_t blk_rounds(Blk<MM>& b, int m) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  int64_t top = 0;
#pragma unroll
  for (int rnd = 0; rnd < 3; rnd++) {
    int64_t c[MM];
    int64_t cout = 0;
#pragma unroll
    for (int j = 0; j < MM; j++) {
      c[j] = 0;
      if (j < m) {
        const int64_t v = b.v[j];
        const int64_t dg = v & kMask;
        c[j] = (v - dg) >> kRadixBits;
        b.v[j] = dg;
        if (j == m - 1) cout = c[j];
      }
    }
    int64_t cin = __shfl_up_sync(full, cout, 1);
    top += __shfl_sync(full, cout, 31);
    if (lane == 0) cin = 0;
#pragma unroll
    for (int j = MM - 1; j >= 1; j--)
      if (j < m) b.v[j] += c[j - 1];
    b.v[0] += cin;
  }
  return top;
}

// resolve pending +1 (sgn > 0: digits >= B generate, == B-1 propagate) or
// -1 (digits < 0 generate, == 0 propagate) carries; returns the signed carry
// that leaves lane 31
template <int MM>
__device__ __forceinline__ int64_t blk_lookahead(Blk<MM>& b, int m, int sgn) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  uint32_t G = 0, P = 0;
#pragma unroll
  for (int j = 0; j < MM; j++) {
    if (j < m) {
      const int64_t v = b.v[j];
      const bool g = sgn > 0 ? (v >= kRadix) : (v < 0);
      const bool pr = sgn > 0 ? (v == kMask) : (v == 0);
      G |= (uint32_t)g << j;
      P |= (uint32_t)pr << j;
    }
  }
  const uint32_t allp = (m >= 32) ? 0xffffffffu : ((1u << m) - 1u);
  auto local = [&](uint32_t cin) -> uint64_t {
    const uint64_t A = ((uint64_t)G << 1) | cin;
    const uint64_t S = (A & P) + P;
    return (S ^ P) | A;  // bit j: carry into digit j; bit m: carry out of the lane
  };
  const uint64_t C0 = local(0);
  const uint32_t Gl = __ballot_sync(full, (C0 >> m) & 1);
  const uint32_t Pl = __ballot_sync(full, P == allp);
  const uint64_t A = ((uint64_t)Gl << 1) & 0xffffffffull;
  const uint64_t S = (A & Pl) + Pl;
  const uint32_t Cin = ((uint32_t)S ^ Pl) | (uint32_t)A;
  const int64_t out31 = (int64_t)(((S >> 32) & 1) | ((Gl >> 31) & 1));
  const uint64_t C = local((Cin >> lane) & 1);
#pragma unroll
  for (int j = 0; j < MM; j++) {
    if (j < m) {
      const int64_t cj = (C >> j) & 1;
      const int64_t oj = ((G >> j) & 1) | (((P >> j) & 1) & cj);
      b.v[j] += sgn > 0 ? (cj - kRadix * oj) : (kRadix * oj - cj);
    }
  }
  return sgn * out31;
}

template <int MM>
__device__ __forceinline__ bool warp_normalize_t(const int64_t* col, int ncols, int drop, int W, int32_t* out) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int m = (ncols + 31) / 32;
  Blk<MM> b;
#pragma unroll
  for (int j = 0; j < MM; j++) {
    const int c = lane * m + j;
    b.v[j] = (j < m && c < ncols) ? col[c] : 0;
    if (drop && c == drop - 1) b.v[j] += kRadix / 2;  // rounding: + B^drop / 2
  }
  int64_t top = blk_rounds(b, m);  // digits in [-1, B]
  top += blk_lookahead(b, m, 1);
  top += blk_lookahead(b, m, -1);  // canonical digits in [0, B), signed carry in `top`
#pragma unroll
  for (int j = 0; j < MM; j++)
    if (lane * m + j < drop) b.v[j] = 0;  // floor: discard the dropped digits
  const bool neg = top < 0;
  if (neg) {
    // |R| = -R: complement the kept digits and add one at column `drop`
#pragma unroll
    for (int j = 0; j < MM; j++) {
      const int c = lane * m + j;
      if (j < m && c >= drop) b.v[j] = kMask - b.v[j] + (c == drop ? 1 : 0);
    }
    top = -top - 1 + blk_lookahead(b, m, 1);
  }
  bool ovf = top != 0;
#pragma unroll
  for (int j = 0; j < MM; j++) {
    const int c = lane * m + j;
    if (j < m && c >= drop) {
      const int d = c - drop;
      const int32_t dig = (int32_t)b.v[j];
      if (d < W)
        out[d] = neg ? -dig : dig;
      else if (dig)
        ovf = true;
    }
  }
  for (int d = 32 * m - drop + lane; d < W; d += 32) out[d] = 0;
  return __any_sync(full, ovf);
}

// ---------------------------------------------------------------------------
// Rounding to balanced semi-normal form (SNF) -- the per-order rounding of the
// recurrence (U_m, coefficient rows, rounded pair sums):
//     digits of rnd(V) = floor((V + B^2/2) / B^2)
// Columns above the top digit position (relative column W+1) are folded into
// it; then three parallel rounds "every column below the top splits into a
// balanced digit in [-B/2, B/2) and a carry round(v/B) that moves one column
// up" leave digits in [-B/2-1, B/2]; the top column absorbs carries and keeps
// the sign. Digit 2 is corrected by floor((d_0 + d_1 B) / B^2). No carry-
// lookahead and no sign conversion: the digits are a deterministic function of
// the exact column value (oracle/fixmodel.c round_cols restates it), they fit
// int32 with |digit| <= B/2 + 2 (except the top one, |top| < B), and small
// values of either sign keep their leading zero digits (zero-digit skipping).
// Canonical digits are only produced for the state (warp_normalize_t, drop 0).
// Overflow: |top digit| >= B.
// Lane layout: M consecutive columns per lane, aligned so that the top column
// topc = W + 1 is the last column of lane 31 (lane l, slot j holds column
// topc - 32 M + 1 + l M + j; columns below 0 are zero). The loop bounds are
// compile-time, so the rounds are straight-line code with M independent
// chains per lane.
template <int M>
__device__ __forceinline__ bool warp_snf_t(const int64_t* col, int ncols, int W, int32_t* out, int2* info) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int topc = W + 1;
  const int c0 = topc - 32 * M + 1 + lane * M;  // column of slot 0
  int64_t v[M];
#pragma unroll
  for (int j = 0; j < M; j++) {
    const int c = c0 + j;
    v[j] = (c >= 0 && c < ncols) ? col[c] : 0;
  }
  if (lane == 31 && ncols > topc + 1) {
    // columns above the top one (fold carries of the column groups) belong to
    // the top digit: v_top += sum_u col[u] B^(u - topc), Horner from the top
    int64_t acc = 0;
    bool big = false;
    for (int u = ncols - 1; u > topc; u--) {
      acc = acc * kRadix + col[u];
      big |= (acc > (int64_t(1) << 34)) || (acc < -(int64_t(1) << 34));
    }
    v[M - 1] = big ? 4 * kRadix : v[M - 1] + acc * kRadix;
  }
  if (c0 <= 1 && c0 + M > 1) {  // rounding: + B^2 / 2
#pragma unroll
    for (int j = 0; j < M; j++)
      if (c0 + j == 1) v[j] += kRadix / 2;
  }
  // rounds 1-2 in 64 bits, round 3 (|v| < 2^29) in 32 bits
#pragma unroll
  for (int rnd = 0; rnd < 2; rnd++) {
    int64_t h[M];
#pragma unroll
    for (int j = 0; j < M; j++) {
      const int64_t t = v[j] + kRadix / 2;
      h[j] = t >> kRadixBits;
      v[j] = (int64_t)(int32_t)(((uint32_t)t & (uint32_t)kMask) - (uint32_t)(kRadix / 2));
    }
    if (lane == 31) {  // the top column absorbs
      v[M - 1] += h[M - 1] * kRadix;
      h[M - 1] = 0;
    }
    int64_t cin = __shfl_up_sync(full, h[M - 1], 1);
    if (lane == 0) cin = 0;
#pragma unroll
    for (int j = M - 1; j >= 1; j--) v[j] += h[j - 1];
    v[0] += cin;
  }
  int32_t w[M];
  {
    int32_t h[M];
#pragma unroll
    for (int j = 0; j < M; j++) {
      const int32_t t = (int32_t)v[j] + (int32_t)(kRadix / 2);
      h[j] = t >> kRadixBits;
      w[j] = (t & (int32_t)kMask) - (int32_t)(kRadix / 2);
    }
    int64_t top = 0;
    if (lane == 31) {
      top = v[M - 1];  // top column keeps its full value
      h[M - 1] = 0;
    }
    int32_t cin = __shfl_up_sync(full, h[M - 1], 1);
    if (lane == 0) cin = 0;
#pragma unroll
    for (int j = M - 1; j >= 1; j--) w[j] += h[j - 1];
    w[0] += cin;
    if (lane == 31) {
      top += (M >= 2 ? h[M - 2 < 0 ? 0 : M - 2] : cin);
      w[M - 1] = (int32_t)(top >= kRadix ? kRadix : (top <= -kRadix ? -kRadix : top));
    }
  }
  // floor((d_0 + d_1 B) / B^2) corrects digit 2 (columns 0, 1, 2 sit in one or two lanes)
  const int p0 = 32 * M - 1 - topc;  // linear slot of column 0
  int32_t s0 = 0, s1 = 0;
#pragma unroll
  for (int j = 0; j < M; j++) {
    if (j == p0 % M) s0 = w[j];
    if (j == (p0 + 1) % M) s1 = w[j];
  }
  const int32_t d0 = __shfl_sync(full, s0, p0 / M);
  const int32_t d1 = __shfl_sync(full, s1, (p0 + 1) / M);
  const int64_t low = (int64_t)d0 + (int64_t)d1 * kRadix;
  const int32_t fix = low < 0 ? -1 : (low >= kRadix * kRadix ? 1 : 0);
  bool ovf = false;
  int bot = 1 << 30, tp = -1;
#pragma unroll
  for (int j = 0; j < M; j++) {
    const int c = c0 + j;
    if (c >= 2) {
      const int d = c - 2;
      const int32_t dig = w[j] + (c == 2 ? fix : 0);
      out[d] = dig;
      if (dig) {
        bot = min(bot, d);
        tp = max(tp, d);
      }
    }
  }
  if (lane == 31 && (w[M - 1] >= kRadix || w[M - 1] <= -kRadix)) ovf = true;
  bot = __reduce_min_sync(full, bot);
  tp = __reduce_max_sync(full, tp);
  if (lane == 0) *info = make_int2(tp >= 0 ? bot : W, tp);
  const bool any = __any_sync(full, ovf);
  __syncwarp();
  return any;
}

__device__ __forceinline__ bool warp_snf(const int64_t* col, int ncols, int W, int32_t* out, int2* info) {
  const int M = (W + 2 + 31) / 32;
  switch (M) {
    case 1: return warp_snf_t<1>(col, ncols, W, out, info);
    case 2: return warp_snf_t<2>(col, ncols, W, out, info);
    case 3: return warp_snf_t<3>(col, ncols, W, out, info);
    case 4: return warp_snf_t<4>(col, ncols, W, out, info);
    case 5: return warp_snf_t<5>(col, ncols, W, out, info);
    case 6: return warp_snf_t<6>(col, ncols, W, out, info);
    case 7: return warp_snf_t<7>(col, ncols, W, out, info);
    case 8: return warp_snf_t<8>(col, ncols, W, out, info);
    case 9: return warp_snf_t<9>(col, ncols, W, out, info);
    case 10: return warp_snf_t<10>(col, ncols, W, out, info);
    case 11: case 12: return warp_snf_t<12>(col, ncols, W, out, info);
    case 13: case 14: case 15: case 16: return warp_snf_t<16>(col, ncols, W, out, info);
    default: return warp_snf_t<kMaxLanesDigits>(col, ncols, W, out, info);
  }
}

// ---------------------------------------------------------------------------
// Group normalisation: NW warps (named barrier `bar_id`, 32*NW threads) share
// one column vector; warp w of the group owns columns [w*32*m, (w+1)*32*m).
// Same algorithm as warp_normalize_t (three parallel carry rounds, then a
// carry-lookahead per sign), with the warp-to-warp carries exchanged through
// the shared scratch `xs` (>= 4*NW + 8 int64). Returns the overflow flag.
__device__ __forceinline__ void group_sync(int bar_id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthreads));
}

template <int MM>
__device__ __forceinline__ int64_t grp_lookahead(Blk<MM>& b, int m, int sgn, int gw, int NW, int bar_id,
                                                 int64_t* xs) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  uint32_t G = 0, P = 0;
#pragma unroll
  for (int j = 0; j < MM; j++) {
    if (j < m) {
      const int64_t v = b.v[j];
      G |= (uint32_t)(sgn > 0 ? (v >= kRadix) : (v < 0)) << j;
      P |= (uint32_t)(sgn > 0 ? (v == kMask) : (v == 0)) << j;
    }
  }
  const uint32_t allp = (m >= 32) ? 0xffffffffu : ((1u << m) - 1u);
  auto local = [&](uint32_t cin) -> uint64_t {
    const uint64_t A = ((uint64_t)G << 1) | cin;
    const uint64_t S = (A & P) + P;
    return (S ^ P) | A;
  };
  const uint64_t C0 = local(0);
  const uint32_t Gl = __ballot_sync(full, (C0 >> m) & 1);
  const uint32_t Pl = __ballot_sync(full, P == allp);
  // warp-level generate / propagate (carry-in 0)
  {
    const uint64_t A = ((uint64_t)Gl << 1) & 0xffffffffull;
    const uint64_t S = (A & Pl) + Pl;
    const int wgen = (int)(((S >> 32) & 1) | ((Gl >> 31) & 1));
    if (lane == 0) {
      xs[2 * gw] = wgen;
      xs[2 * gw + 1] = (Pl == full) ? 1 : 0;
    }
  }
  group_sync(bar_id, 32 * NW);
  int wcin = 0;
  for (int w = 0; w < gw; w++) wcin = (int)xs[2 * w] | ((int)xs[2 * w + 1] & wcin);
  int gout = 0;  // carry leaving the last warp
  {
    int cc = 0;
    for (int w = 0; w < NW; w++) cc = (int)xs[2 * w] | ((int)xs[2 * w + 1] & cc);
    gout = cc;
  }
  const uint64_t A = (((uint64_t)Gl << 1) | (uint64_t)wcin) & 0xffffffffull;
  const uint64_t S = (A & Pl) + Pl;
  const uint32_t Cin = ((uint32_t)S ^ Pl) | (uint32_t)A;
  const uint64_t C = local((Cin >> lane) & 1);
#pragma unroll
  for (int j = 0; j < MM; j++) {
    if (j < m) {
      const int64_t cj = (C >> j) & 1;
      const int64_t oj = ((G >> j) & 1) | (((P >> j) & 1) & cj);
      b.v[j] += sgn > 0 ? (cj - kRadix * oj) : (kRadix * oj - cj);
    }
  }
  group_sync(bar_id, 32 * NW);  // xs reused by the next step
  return sgn * (int64_t)gout;
}

template <int MM>
__device__ __forceinline__ bool group_normalize_t(const int64_t* col, int ncols, int drop, int W, int32_t* out,
                                                  int gw, int NW, int bar_id, int64_t* xs) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int per = (ncols + 32 * NW - 1) / (32 * NW);  // m: columns per lane
  const int m = per;
  const int base = gw * 32 * m;
  Blk<MM> b;
#pragma unroll
  for (int j = 0; j < MM; j++) {
    const int c = base + lane * m + j;
    b.v[j] = (j < m && c < ncols) ? col[c] : 0;
    if (drop && c == drop - 1) b.v[j] += kRadix / 2;
  }
  int64_t top = 0;
#pragma unroll
  for (int rnd = 0; rnd < 3; rnd++) {
    int64_t c[MM];
    int64_t cout = 0;
#pragma unroll
    for (int j = 0; j < MM; j++) {
      c[j] = 0;
      if (j < m) {
        const int64_t v = b.v[j];
        const int64_t dg = v & kMask;
        c[j] = (v - dg) >> kRadixBits;
        b.v[j] = dg;
        if (j == m - 1) cout = c[j];
      }
    }
    int64_t cin = __shfl_up_sync(full, cout, 1);
    const int64_t wout = __shfl_sync(full, cout, 31);
    if (lane == 0) xs[2 * gw] = wout;
    group_sync(bar_id, 32 * NW);
    if (lane == 0) cin = gw > 0 ? xs[2 * (gw - 1)] : 0;
    top += xs[2 * (NW - 1)];
#pragma unroll
    for (int j = MM - 1; j >= 1; j--)
      if (j < m) b.v[j] += c[j - 1];
    b.v[0] += cin;
    group_sync(bar_id, 32 * NW);
  }
  top += grp_lookahead(b, m, 1, gw, NW, bar_id, xs);
  top += grp_lookahead(b, m, -1, gw, NW, bar_id, xs);
#pragma unroll
  for (int j = 0; j < MM; j++)
    if (base + lane * m + j < drop) b.v[j] = 0;
  const bool neg = top < 0;  // uniform over the group
  if (neg) {
#pragma unroll
    for (int j = 0; j < MM; j++) {
      const int c = base + lane * m + j;
      if (j < m && c >= drop) b.v[j] = kMask - b.v[j] + (c == drop ? 1 : 0);
    }
    top = -top - 1 + grp_lookahead(b, m, 1, gw, NW, bar_id, xs);
  }
  bool ovf = top != 0;
#pragma unroll
  for (int j = 0; j < MM; j++) {
    const int c = base + lane * m + j;
    if (j < m && c >= drop) {
      const int d = c - drop;
      const int32_t dig = (int32_t)b.v[j];
      if (d < W)
        out[d] = neg ? -dig : dig;
      else if (dig)
        ovf = true;
    }
  }
  for (int d = 32 * NW * m - drop + gw * 32 + lane; d < W; d += 32 * NW) out[d] = 0;
  ovf = __any_sync(full, ovf);
  if (lane == 0) xs[2 * gw] = ovf ? 1 : 0;
  group_sync(bar_id, 32 * NW);
  bool any = false;
  for (int w = 0; w < NW; w++) any |= xs[2 * w] != 0;
  group_sync(bar_id, 32 * NW);
  return any;
}

// group normalisation + bot/top info (+ optional rounding to prec bits by warp 0)
static __device__ __noinline__ bool group_normalize(const int64_t* col, int ncols, int drop, int W, int32_t* out,
                                             int2* info, int round_prec_bits, int gw, int NW, int bar_id,
                                             int64_t* xs);

__device__ inline void round_to_prec(int32_t* out, int W, int prec_bits, bool& ovf) {
  // lane-0 sequential: round the canonical digit vector to prec_bits
  // significant bits, ties to even (the reference's state precision).
  int tp = -1;
  for (int d = W - 1; d >= 0; d--)
    if (out[d]) {
      tp = d;
      break;
    }
  if (tp < 0) return;
  const bool neg = out[tp] < 0;
  auto mag = [&](int d) -> int32_t { return out[d] < 0 ? -out[d] : out[d]; };
  const int nbits = kRadixBits * tp + (32 - __clz(mag(tp)));
  const int s = nbits - prec_bits;  // number of low bits to drop
  if (s <= 0) return;
  const int sd = s / kRadixBits, sb = s % kRadixBits;
  const int hp = s - 1, hd = hp / kRadixBits, hb = hp % kRadixBits;
  const bool half = (mag(hd) >> hb) & 1;
  const bool lsb = (mag(sd) >> sb) & 1;
  bool sticky = (mag(hd) & ((1 << hb) - 1)) != 0;
  for (int d = 0; d < hd && !sticky; d++) sticky = out[d] != 0;
  for (int d = 0; d < sd; d++) out[d] = 0;
  int64_t m = mag(sd) & ~((int64_t(1) << sb) - 1);
  int64_t cin = (half && (sticky || lsb)) ? (int64_t(1) << sb) : 0;
  for (int d = sd; d < W; d++) {
    if (d > sd) {
      if (!cin) break;
      m = mag(d);
    }
    m += cin;
    cin = m >> kRadixBits;
    m &= kMask;
    out[d] = (int32_t)(neg ? -m : m);
  }
  if (cin) ovf = true;
}

template <int MAXM>
__device__ __forceinline__ bool warp_normalize_upto(const int64_t* col, int ncols, int drop, int W, int32_t* out,
                                                int2* info, int round_prec_bits);

__device__ __forceinline__ bool warp_normalize(const int64_t* col, int ncols, int drop, int W, int32_t* out, int2* info,
                                      int round_prec_bits) {
  return warp_normalize_upto<kMaxLanesDigits>(col, ncols, drop, W, out, info, round_prec_bits);
}

// ncols <= 256 (<= 8 digits per lane): fewer instantiations, fewer registers
__device__ __forceinline__ bool warp_normalize_small(const int64_t* col, int ncols, int drop, int W, int32_t* out,
                                                     int2* info, int round_prec_bits) {
  return warp_normalize_upto<8>(col, ncols, drop, W, out, info, round_prec_bits);
}

template <int MAXM>
__device__ __forceinline__ bool warp_normalize_upto(const int64_t* col, int ncols, int drop, int W, int32_t* out,
                                                int2* info, int round_prec_bits) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int m = (ncols + 31) / 32;
  if (drop == 2 && round_prec_bits == 0) return warp_snf(col, ncols, W, out, info);
  bool ovf;
  if (m <= 2)
    ovf = warp_normalize_t<2>(col, ncols, drop, W, out);
  else if (m <= 4)
    ovf = warp_normalize_t<4>(col, ncols, drop, W, out);
  else if (MAXM <= 8 || m <= 8)
    ovf = warp_normalize_t<(MAXM < 8 ? MAXM : 8)>(col, ncols, drop, W, out);
  else if (MAXM <= 16 || m <= 16)
    ovf = warp_normalize_t<(MAXM < 16 ? MAXM : 16)>(col, ncols, drop, W, out);
  else
    ovf = warp_normalize_t<MAXM>(col, ncols, drop, W, out);
  __syncwarp();
  if (round_prec_bits > 0) {
    if (lane == 0) round_to_prec(out, W, round_prec_bits, ovf);
    ovf = __shfl_sync(full, ovf, 0);
    __syncwarp();
  }
  int bot = 1 << 30, tp = -1;
  for (int d = lane; d < W; d += 32)
    if (out[d]) {
      bot = min(bot, d);
      tp = max(tp, d);
    }
  bot = __reduce_min_sync(full, bot);
  tp = __reduce_max_sync(full, tp);
  if (lane == 0) *info = make_int2(tp >= 0 ? bot : W, tp);
  __syncwarp();
  return ovf;
}

static __device__ __noinline__ bool group_normalize(const int64_t* col, int ncols, int drop, int W, int32_t* out,
                                             int2* info, int round_prec_bits, int gw, int NW, int bar_id,
                                             int64_t* xs) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int m = (ncols + 32 * NW - 1) / (32 * NW);
  if (drop == 2 && round_prec_bits == 0) {  // SNF: one warp of the group, the others wait
    if (gw == 0 && warp_snf(col, ncols, W, out, info) && lane == 0) xs[0] = 1;
    else if (gw == 0 && lane == 0) xs[0] = 0;
    group_sync(bar_id, 32 * NW);
    const bool o = xs[0] != 0;
    group_sync(bar_id, 32 * NW);
    return o;
  }
  bool ovf;
  if (m <= 2)
    ovf = group_normalize_t<2>(col, ncols, drop, W, out, gw, NW, bar_id, xs);
  else if (m <= 4)
    ovf = group_normalize_t<4>(col, ncols, drop, W, out, gw, NW, bar_id, xs);
  else if (m <= 8)
    ovf = group_normalize_t<8>(col, ncols, drop, W, out, gw, NW, bar_id, xs);
  else
    ovf = group_normalize_t<16>(col, ncols, drop, W, out, gw, NW, bar_id, xs);
  if (round_prec_bits > 0) {
    group_sync(bar_id, 32 * NW);
    if (gw == 0 && lane == 0) round_to_prec(out, W, round_prec_bits, ovf);
    if (gw == 0 && lane == 0) xs[0] = ovf ? 1 : 0;
    group_sync(bar_id, 32 * NW);
    ovf = xs[0] != 0;
    group_sync(bar_id, 32 * NW);
  }
  int bot = 1 << 30, tp = -1;
  for (int d = gw * 32 + lane; d < W; d += 32 * NW)
    if (out[d]) {
      bot = min(bot, d);
      tp = max(tp, d);
    }
  bot = __reduce_min_sync(full, bot);
  tp = __reduce_max_sync(full, tp);
  if (lane == 0) {
    xs[2 * gw] = bot;
    xs[2 * gw + 1] = tp;
  }
  group_sync(bar_id, 32 * NW);
  if (gw == 0 && lane == 0) {
    int B0 = 1 << 30, T0 = -1;
    for (int w = 0; w < NW; w++) {
      B0 = min(B0, (int)xs[2 * w]);
      T0 = max(T0, (int)xs[2 * w + 1]);
    }
    *info = make_int2(T0 >= 0 ? B0 : W, T0);
  }
  group_sync(bar_id, 32 * NW);
  return ovf;
}

// ---------------------------------------------------------------------------
// Folded partial units: a thread's (column group, operand slice) accumulator
// is stored as kR uint32 digits (relative columns c0-T .. c0-T+kR-1) plus the
// group's outgoing carry; a column's total over n units u0, u0+ustride, ... is
// the digits of the group owning it plus the carry of the group below.
__device__ __forceinline__ void unit_store(uint32_t* part, int64_t* pcar, const Acc& a, int grp, int c0, int T) {
#pragma unroll
  for (int r = 0; r < kR; r++) {
    const int c = c0 + r - T;
    if (c >= 0) part[c] = (uint32_t)a.v[r];
  }
  pcar[grp] = a.v[kR];
}

__device__ __forceinline__ int64_t unit_column(const uint32_t* part, const int64_t* pcar, int u0, int ustride, int n,
                                               int ncx, int ngstride, int c, int T, int gf, int ng) {
  const int cabs = c + T;
  const int own = cabs / kR - gf;
  const int cgb = (cabs % kR == 0) ? cabs / kR - 1 - gf : -1;
  int64_t s = 0;
  if (own >= 0 && own < ng) {
    const uint32_t* pp = part + (size_t)u0 * ncx + c;
#pragma unroll 4
    for (int u = 0; u < n; u++) s += pp[(size_t)u * ustride * ncx];
  }
  if (cgb >= 0 && cgb < ng) {
    const int64_t* pc = pcar + (size_t)u0 * ngstride + cgb;
#pragma unroll 4
    for (int u = 0; u < n; u++) s += pc[(size_t)u * ustride * ngstride];
  }
  return s;
}

}  // namespace mpt
