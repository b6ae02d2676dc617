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
  int64_t d;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
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

// ---------------------------------------------------------------------------
// Warp-cooperative normalisation of a column vector (relative columns
// 0..ncols-1, value V = sum col[c] B^c, |col[c]| < 2^62) into canonical signed
// digits of floor((V + [drop] B^drop / 2) / B^drop), drop in {0, 2}.
// Lane l holds columns [l*m, l*m+m). Carries are resolved without
// data-dependent loops: one local pass, two shuffle passes (carries shrink to
// {-1, 0, +1}), then a ballot carry-lookahead per sign:
//   carry-in mask C = (((A & P) + P) ^ P) | A,  A = lanes receiving a carry,
//   P = lanes whose block would pass it on (all digits B-1, or all 0 for borrows).
template <int MM>
struct Blk {
  int64_t v[MM];
};

// add `cin` to the block (digit 0 upward); digits back to [0, B); returns carry out
template <int MM>
__device__ __forceinline__ int64_t blk_add(Blk<MM>& b, int m, int64_t cin) {
#pragma unroll
  for (int j = 0; j < MM; j++) {
    if (j < m) {
      const int64_t t = b.v[j] + cin;
      const int64_t dgt = t & kMask;
      cin = (t - dgt) >> kRadixBits;
      b.v[j] = dgt;
    }
  }
  return cin;
}

template <int MM>
__device__ __forceinline__ bool blk_all(const Blk<MM>& b, int m, int64_t val) {
  bool all = true;
#pragma unroll
  for (int j = 0; j < MM; j++)
    if (j < m) all &= (b.v[j] == val);
  return all;
}

// resolve pending carries e (from this lane into the next) in {-1, 0, 1};
// `top` collects what leaves lane 31
template <int MM>
__device__ __forceinline__ void blk_resolve(Blk<MM>& b, int m, int e, int64_t& top) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int ein = __shfl_up_sync(full, e, 1);
  const int e31 = __shfl_sync(full, e, 31);
  top += e31;
#pragma unroll
  for (int sgn = 1; sgn >= -1; sgn -= 2) {
    const unsigned A = __ballot_sync(full, lane > 0 && ein == sgn);
    const unsigned P = __ballot_sync(full, blk_all(b, m, sgn > 0 ? kMask : 0));
    const unsigned long long S = (unsigned long long)(A & P) + P;
    const unsigned C = ((unsigned)S ^ P) | A;
    top += sgn * (int64_t)(S >> 32);
    if ((C >> lane) & 1u) blk_add(b, m, sgn);
  }
}

template <int MM>
__device__ __forceinline__ void blk_carry(Blk<MM>& b, int m, int64_t& top) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  int64_t c = blk_add(b, m, 0);
#pragma unroll
  for (int pass = 0; pass < 2; pass++) {
    int64_t cin = __shfl_up_sync(full, c, 1);
    top += __shfl_sync(full, c, 31);
    if (lane == 0) cin = 0;
    c = blk_add(b, m, cin);
  }
  blk_resolve(b, m, (int)c, top);
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
  int64_t top = 0;
  blk_carry(b, m, top);  // digits in [0, B), signed carry in `top`
  if (drop) {
#pragma unroll
    for (int j = 0; j < MM; j++)
      if (lane * m + j < drop) b.v[j] = 0;  // floor: discard the low digits
  }
  if (false) {
    // + B^drop / 2 == + B/2 at column drop-1, then floor: discard columns < drop
    int e = 0;
    if (lane * m <= drop - 1 && drop - 1 < lane * m + m) {
      int64_t cin = 0;
#pragma unroll
      for (int j = 0; j < MM; j++) {
        if (j < m) {
          const int64_t t = b.v[j] + cin + ((lane * m + j == drop - 1) ? (kRadix / 2) : 0);
          const int64_t dgt = t & kMask;
          cin = (t - dgt) >> kRadixBits;
          b.v[j] = dgt;
        }
      }
      e = (int)cin;
    }
    blk_resolve(b, m, e, top);
#pragma unroll
    for (int j = 0; j < MM; j++)
      if (lane * m + j < drop) b.v[j] = 0;
  }
  const bool neg = top < 0;
  if (neg) {
    // |R| = -R: complement the kept digits and add one at column `drop`
    int e = 0;
#pragma unroll
    for (int j = 0; j < MM; j++)
      if (j < m && lane * m + j >= drop) b.v[j] = kMask - b.v[j];
    top = -top - 1;
    if (lane * m <= drop && drop < lane * m + m) {
      int64_t cin = 0;
#pragma unroll
      for (int j = 0; j < MM; j++) {
        if (j < m) {
          const int64_t t = b.v[j] + cin + ((lane * m + j == drop) ? 1 : 0);
          const int64_t dgt = t & kMask;
          cin = (t - dgt) >> kRadixBits;
          b.v[j] = dgt;
        }
      }
      e = (int)cin;
    }
    blk_resolve(b, m, e, top);
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

}  // namespace mpt
