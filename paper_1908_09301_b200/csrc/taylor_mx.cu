// Matrix-recurrence kernel ("mx"): one trajectory per thread-block cluster of
// G = 2..16 CTAs (sm_100a); the per-order critical path runs on CTA 0 ("lead").
//
// Arithmetic (restated bit for bit by oracle/fixmodel.c jet_mx): with
// a~_{i+1} = C_i U_i (C_i = tau/(i+1): the tau-scaled rows of the reference's
// taylor.py:117 _jet_rows) the numerator of order j = i+1 is linear in U_i
// apart from the Cauchy sums, which split into the lag-1 terms (rows j-1 and
// 1) and the rest L'(j) (rows 2..j-2):
//
//   U_j   = rnd( sum_j' U_i^j' (x) K_i^{m,j'} + sum_t q_t [lag_t(j) + sum_o split1(P_{o,t}(j))] )
//   K_i   = rnd( S (x) C_i ),   S^{m,j'} = bnf(lin[m][j'] + sum_t q_t a~_0)     (per step, bulk CTAs)
//   a~_j  = rnd( U_i (x) C_i )
//
// The lead computes, per order, every product of U_i, the new coefficient
// rows and the lag-1 terms -- one warp per product, all in parallel -- and
// one rounding per output. The bulk CTAs (ranks 1..G-1, owner of k =
// 1+(k-1) mod (G-1)) receive each new row from the lead and compute their
// share of L'(j) two orders ahead, so DSMEM latency and their work are off
// the critical path. Products are exact int64 column sums (every operand
// digit is balanced or semi-normal, so no folds are needed), hence the cheap
// semi-normal rounding (warp_snf_t) is a deterministic function of the
// inputs and the CPU model reproduces it bit for bit.
//
// Work mapping of one product on one warp: the 8-column groups g and
// ng-1-g are paired (balanced work), each pair's p-range is split evenly over
// NCH consecutive lanes; a lane runs an 8-column register window (one LDS of
// A and one of B per 8 IMAD.WIDE); the NCH lanes then reduce-scatter their 16
// partial columns with shuffles and store exact column sums.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "mpt_common.cuh"
#include "mpt_device.cuh"

namespace cg = cooperative_groups;

namespace mpt {
namespace mx {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kMacWarps = kWarps - 1;  // warp 15 of the lead gathers L'
constexpr int kMaxProd = 32;           // products per lead stage
constexpr int kPerWarpPass = 4;        // bulk products accumulated per lane before a split
constexpr int kQ = 16;                 // zero-skipping width quantum (digits)
constexpr int kMaxQ = 4;               // widths up to 64 digits (K <= ~500): 2 x 4 x 4 product shapes
constexpr int kShapes = 2 * kMaxQ * kMaxQ;
constexpr int kScrStride = 33;         // int64 per column of a warp's window scratch (32 lanes + 1: bank spread)

struct Geo {
  int W, KW, T, Tc, ncols, ncp, ng, rs, krs, urs;
};

__host__ __device__ inline Geo make_geo(const Params& p) {
  Geo g;
  g.W = p.W;
  g.KW = p.W + 1;
  g.T = p.Lf - 2;
  g.Tc = p.Lf + p.sc - 2;
  g.ncols = p.Lf + 4;              // relative columns of every column vector (oracle: ncols)
  g.ncp = (g.ncols + 3) / 4 * 4;
  g.ng = (p.Lf + 3 + 7) / 8;       // 8-column groups covering every product column (rel. <= Lf+2)
  g.rs = (g.KW + 3) / 4 * 4 + kPad;
  g.krs = (g.KW + 3) / 4 * 4;
  g.urs = (g.W + 3) / 4 * 4;
  return g;
}

__host__ __device__ inline int nch_for(const Geo& g) {
  const int np = (g.ng + 1) / 2;
  return np <= 2 ? 16 : np <= 4 ? 8 : np <= 8 ? 4 : 2;
}
__host__ __device__ inline int snf_m(int Wout) { return (Wout + 2 + 31) / 32; }

// active entries (m, j) of the K matrix; dyn: depends on the state (bilinear)
__host__ __device__ inline int n_entries(const Params& p, int* em, int* ej, int* dyn = nullptr) {
  int n = 0;
  for (int m = 0; m < p.D; m++)
    for (int j = 0; j < p.D; j++) {
      const bool lin = !(p.lin_small[m * p.D + j] && p.lin_int[m * p.D + j] == 0);
      bool bil = false;
      for (int t = 0; t < p.NT; t++)
        if (p.teq[t] == m && (p.pj[p.tpair[t]] == j || p.pk[p.tpair[t]] == j)) bil = true;
      if (lin || bil) {
        if (em) em[n] = m;
        if (ej) ej[n] = j;
        if (dyn) dyn[n] = bil;
        n++;
      }
    }
  return n;
}

struct Layout {
  int Gb, nE, nslots;
  size_t off_lrow, off_linfo, off_cpart, off_lsum, off_cbuf, off_recv, off_ssum, off_cinf, off_scr, off_lshr, off_lshg,
      lead_total;
  size_t off_rows, off_rinfo, off_srow, off_sinfo, off_crow, off_cinfo, off_wcol, off_acc, off_bcc, off_kst,
      off_kcol, off_bscr, off_bshr, off_bshg, bulk_total;
  size_t total;
};

// bulk row store: left-hand pair variables for every k, the others for the owned
// class only. Returns the first slot of variable v (v = -1: total), full[v].
__host__ __device__ inline int row_slots(const Params& p, int G, int v, int* full) {
  const int Gb = G - 1;
  int s = 0;
  for (int u = 0; u < p.D; u++) {
    int is_left = 0;
    for (int q = 0; q < p.NP; q++) is_left |= (p.pj[q] == u);
    const int f = is_left || Gb <= 1;
    if (u == v) {
      if (full) *full = f;
      return s;
    }
    s += f ? p.N + 1 : p.N / (Gb > 0 ? Gb : 1) + 2;
  }
  return s;
}

// lead rows: ST D | SB D | LIN D*D | U 2D | K 2nE | C 2 | ROW 2D | ROW1 D
__host__ __device__ inline Layout make_layout(const Params& p, int G) {
  Layout L;
  const Geo g = make_geo(p);
  L.Gb = G - 1;
  L.nE = n_entries(p, nullptr, nullptr);
  const int NPp = p.NP > 0 ? p.NP : 1;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o += (bytes + 15) / 16 * 16;
    return r;
  };
  const int nlrow = 2 * p.D + p.D * p.D + 2 * p.D + 2 * L.nE + 2 + 3 * p.D;
  L.off_lrow = take(sizeof(int32_t) * ((size_t)nlrow * g.rs + 3 * kPad));
  L.off_linfo = take(sizeof(int2) * (size_t)nlrow);
  L.off_cpart = take(sizeof(int64_t) * (size_t)kMaxProd * g.ncp);
  L.off_lsum = take(sizeof(int64_t) * (size_t)kMaxD * g.ncp);
  L.off_cbuf = take(sizeof(int64_t) * (size_t)2 * kMaxD * g.ncp);
  L.off_recv = take(sizeof(int64_t) * 2 * (size_t)(L.Gb > 0 ? L.Gb : 1) * NPp * g.ncp);
  L.off_ssum = take(sizeof(int64_t) * (size_t)p.D * (g.W + 3));
  L.off_cinf = take(sizeof(int2) * (size_t)p.N);
  L.off_scr = take(sizeof(int64_t) * (size_t)kWarps * kScrStride * 8);
  L.off_lshr = take(0);
  L.off_lshg = take(0);
  L.lead_total = o;
  o = 0;
  L.nslots = row_slots(p, G, -1, nullptr) + p.D;  // + row 2 of every variable (the k = 2 Cauchy terms)
  L.off_rows = take(sizeof(int32_t) * ((size_t)L.nslots * g.rs + 3 * kPad));
  L.off_rinfo = take(sizeof(int2) * (size_t)L.nslots);
  L.off_srow = take(sizeof(int32_t) * ((size_t)p.D * p.D * g.rs + 2 * kPad));
  L.off_sinfo = take(sizeof(int2) * (size_t)p.D * p.D);
  L.off_crow = take(sizeof(int32_t) * ((size_t)g.rs + 2 * kPad));
  L.off_cinfo = take(sizeof(int2) * 2);
  L.off_wcol = take(sizeof(int64_t) * (size_t)kWarps * g.ncp);
  L.off_acc = take(sizeof(int64_t) * (size_t)NPp * g.ncp);
  L.off_bcc = take(sizeof(int64_t) * (size_t)NPp * g.ncp);
  L.off_kst = take(sizeof(int32_t) * (size_t)kWarps * g.krs);
  L.off_kcol = take(sizeof(int64_t) * (size_t)kWarps * g.ncp);
  L.off_bscr = take(sizeof(int64_t) * (size_t)kWarps * kScrStride * 8);
  L.off_bshr = take(0);
  L.off_bshg = take(0);
  L.bulk_total = o;
  L.total = L.lead_total > L.bulk_total ? L.lead_total : L.bulk_total;
  return L;
}

// ---------------------------------------------------------------------------
// mbarrier / st.async helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n .reg .pred p;\n MXW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra MXW;\n}" ::"r"(smem_u32(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void st_async16(uint32_t raddr, int32_t a, int32_t b, int32_t c, int32_t d, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];" ::"r"(raddr),
               "r"(a), "r"(b), "r"(c), "r"(d), "r"(rbar)
               : "memory");
}
// one TMA bulk copy from this CTA's shared memory into another CTA's (cluster
// address from mapa), completing `bytes` on the destination's mbarrier
__device__ __forceinline__ void bulk_push(uint32_t rdst, uint32_t lsrc, uint32_t bytes, uint32_t rbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(rdst),
      "r"(lsrc), "r"(bytes), "r"(rbar)
      : "memory");
}
// one TMA bulk copy from global memory into the same shared offset of every CTA
// in `mask` (cluster ranks), completing `bytes` on each one's mbarrier (same offset)
__device__ __forceinline__ void bulk_multicast(uint32_t ldst, const void* gsrc, uint32_t bytes, uint32_t lbar,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
          ldst),
      "l"(gsrc), "r"(bytes), "r"(lbar), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_barrier() {
  cluster_arrive_release();
  cluster_wait_acquire();
}

// ---------------------------------------------------------------------------
// Value-exact balanced digits of V = sum val[c] B^c (oracle bnf_exact): the
// balanced rounding of col' = (-B/2, 0, val...), i.e. warp_bnf_t below with
// the rounding half cancelled.
template <int M>
__device__ __forceinline__ uint64_t la_carries(uint32_t G, uint32_t P) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const uint32_t allp = (M >= 32) ? 0xffffffffu : ((1u << M) - 1u);
  auto local = [&](uint32_t cin) -> uint64_t {
    const uint64_t A = ((uint64_t)G << 1) | cin;
    const uint64_t S = (A & P) + P;
    return (S ^ P) | A;
  };
  const uint64_t C0 = local(0);
  const uint32_t Gl = __ballot_sync(full, (C0 >> M) & 1);
  const uint32_t Pl = __ballot_sync(full, P == allp);
  const uint64_t A = ((uint64_t)Gl << 1) & 0xffffffffull;
  const uint64_t S = (A & Pl) + Pl;
  const uint32_t Cin = ((uint32_t)S ^ Pl) | (uint32_t)A;
  return local((Cin >> lane) & 1);
}

// balanced rounding R = floor((V + B^2/2)/B^2) with every digit in [-B/2, B/2)
// (oracle round_bnf); col[c] for c < ncols, lane l holds columns l*M..l*M+M-1
template <int M>
__device__ __noinline__ bool warp_bnf(const int64_t* col, int ncols, int Wout, int32_t* out, int2* info) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  Blk<M> b;
#pragma unroll
  for (int j = 0; j < M; j++) {
    const int c = lane * M + j;
    b.v[j] = c < ncols ? col[c] : 0;
    if (c == 1) b.v[j] += kRadix / 2;
  }
  int64_t top = blk_rounds(b, M);
  top += blk_lookahead(b, M, 1);
  top += blk_lookahead(b, M, -1);
  const int topc = Wout + 1;
  bool nz = false, nmax = false;
#pragma unroll
  for (int j = 0; j < M; j++) {
    const int c = lane * M + j;
    if (c > topc) {
      nz |= b.v[j] != 0;
      nmax |= b.v[j] != kMask;
    }
  }
  const bool anynz = __any_sync(full, nz), anynmax = __any_sync(full, nmax);
  int64_t hi = 0;
  bool ovf = false;
  if (!anynz && top == 0)
    hi = 0;
  else if (!anynmax && top == -1)
    hi = -1;
  else
    ovf = true;
  uint32_t G = 0, P = 0;
#pragma unroll
  for (int j = 0; j < M; j++) {
    const int c = lane * M + j;
    if (c >= 2 && c < topc) {
      G |= (uint32_t)(b.v[j] >= kRadix / 2) << j;
      P |= (uint32_t)(b.v[j] == kRadix / 2 - 1) << j;
    }
  }
  const uint64_t C = la_carries<M>(G, P);
  int bot = 1 << 30, tp = -1;
#pragma unroll
  for (int j = 0; j < M; j++) {
    const int c = lane * M + j;
    if (c >= 2 && c <= topc) {
      const int64_t cin = (C >> j) & 1;
      int64_t e;
      if (c < topc) {
        const int64_t cout = ((G >> j) & 1) | (((P >> j) & 1) & cin);
        e = b.v[j] + cin - kRadix * cout;
      } else {
        e = b.v[j] + cin + hi * kRadix;
        if (e >= kRadix / 2 || e < -(kRadix / 2)) ovf = true;
      }
      const int d = c - 2;
      out[d] = (int32_t)e;
      if (e) {
        bot = min(bot, d);
        tp = max(tp, d);
      }
    }
  }
  bot = __reduce_min_sync(full, bot);
  tp = __reduce_max_sync(full, tp);
  if (lane == 0 && info) *info = make_int2(tp >= 0 ? bot : Wout, tp);
  const bool any = __any_sync(full, ovf);
  __syncwarp();
  return any;
}

// semi-normal rounding of exact column sums (oracle round_cols), one warp
template <int M>
__device__ __noinline__ bool warp_snf_call(const int64_t* col, int ncols, int W, int32_t* out, int2* info) {
  return warp_snf_t<M>(col, ncols, W, out, info);
}

__device__ __noinline__ bool warp_canon(const int64_t* col, int ncols, int W, int32_t* out, int2* info, int prec) {
  return warp_normalize(col, ncols, 0, W, out, info, prec);
}

// ---------------------------------------------------------------------------
// exact products on one warp

// s64 += s32 * s32 as one IMAD.WIDE (the C++ form lets nvcc split it into
// IMAD.WIDE.U32 + sign corrections)
__device__ __forceinline__ int64_t madw(int32_t a, int32_t b, int64_t c) {
  int64_t d;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}
// shared-memory accesses by 32-bit address (used inside the out-of-line product
// routine, where the data is stable for the whole call)
__device__ __forceinline__ int32_t lds32(uint32_t a) {
  int32_t v;
  asm("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int64_t lds64(uint32_t a) {
  int64_t v;
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts64(uint32_t a, int64_t v) {
  asm volatile("st.shared.b64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}

// one masked chunk of 4 p-steps: acc[r] += sum_{p in [p0, min(p0+3, p1)]} A[p] B[c0+r-p]
__device__ __forceinline__ void mac_chunk4(int64_t (&acc)[8], uint32_t A, uint32_t B, int c0, int p0, int p1) {
  int32_t a[4], b[11];
#pragma unroll
  for (int u = 0; u < 4; u++) a[u] = (p0 + u <= p1) ? lds32(A + 4 * (p0 + u)) : 0;
#pragma unroll
  for (int t = 0; t < 11; t++) b[t] = lds32(B + 4 * (c0 - p0 - 3 + t));  // b[t] = B[c0 - p0 - 3 + t]
#pragma unroll
  for (int u = 0; u < 4; u++)
#pragma unroll
    for (int r = 0; r < 8; r++) acc[r] = madw(a[u], b[r - u + 3], acc[r]);
}

// acc += sum_{p in [p0, p1]} A[p] B[c0+r-p]: one p-step per iteration (8
// IMAD.WIDE on the 8-column window, no masked work), next operands loaded one
// step ahead; rows are zero-padded, so the look-ahead reads are harmless
__device__ __forceinline__ void mac_run(int64_t (&acc)[8], uint32_t A, uint32_t B, int c0, int p0, int p1) {
#if MX_MAC_CHUNK4
#pragma unroll 1
  for (int q = p0; q <= p1; q += 4) mac_chunk4(acc, A, B, c0, q, p1);
#else
  if (p0 > p1) return;
  int32_t w[8];
#pragma unroll
  for (int r = 0; r < 8; r++) w[r] = lds32(B + 4 * (c0 + r - p0));
  int32_t a = lds32(A + 4 * p0), bn = lds32(B + 4 * (c0 - p0 - 1));
#pragma unroll 2
  for (int p = p0; p <= p1; p++) {
    const int32_t an = lds32(A + 4 * (p + 1)), bnn = lds32(B + 4 * (c0 - p - 2));
#pragma unroll
    for (int r = 0; r < 8; r++) acc[r] = madw(a, w[r], acc[r]);
#pragma unroll
    for (int r = 7; r > 0; r--) w[r] = w[r - 1];
    w[0] = bn;
    a = an;
    bn = bnn;
  }
#endif
}

// one masked block of 8 p-steps: acc[r] += sum_{p in [p0, min(p0+7, p1)]} A[p] B[c0+r-p];
// straight-line code (8 loads of A, 15 of B, 64 IMAD.WIDE). Rows are zero-padded
// by kPad digits, so the reads past the ranges are harmless.
__device__ __forceinline__ void mac_block(int64_t (&acc)[8], uint32_t A, uint32_t B, int c0, int p0, int p1) {
  int32_t a[8], b[15];
#pragma unroll
  for (int u = 0; u < 8; u++) a[u] = (p0 + u <= p1) ? lds32(A + 4 * (p0 + u)) : 0;
#pragma unroll
  for (int t = 0; t < 15; t++) b[t] = lds32(B + 4 * (c0 - p0 - 7 + t));
#pragma unroll
  for (int u = 0; u < 8; u++)
#pragma unroll
    for (int r = 0; r < 8; r++) acc[r] = madw(a[u], b[r - u + 7], acc[r]);
}

// useful digit products of group [c0, c0+8) for nonzero ranges ia, ib (counters only)
__device__ __forceinline__ unsigned long long group_macs(int2 ia, int2 ib, int c0) {
  unsigned long long n = 0;
  for (int r = 0; r < 8; r++) {
    const int c = c0 + r;
    const int lo = max(ia.x, c - ib.y), hi = min(ia.y, c - ib.x);
    if (hi >= lo) n += hi - lo + 1;
  }
  return n;
}

// A product for the out-of-line warp routine: shared addresses of digit 0 of
// both rows and their nonzero ranges.
struct Prod {
  uint32_t A, B;
  int2 ia, ib;
};

// One warp: sum_k A_k (x) B_k (truncation T, relative column c - T), nprod <=
// 4 products accumulated exactly in the lanes' registers, then the NCH lanes
// of each group pair reduce-scatter and the exact columns are stored to
// `out` (shared address of int64[nout+...]): overwritten (zero-filled first)
// or accumulated. Group pairs (g, ng-1-g) balance the triangle; blocks of 8
// p-steps are dealt round-robin to the pair's lanes. ONE out-of-line copy of
// this code serves every product of the kernel (instruction-cache footprint).
template <int NCH>
__device__ __noinline__ void warp_prods(const Prod* desc, int nprod, int T, int ng, uint32_t out, int ncp, int nout,
                                        int accumulate, MacCount* mc) {
  const int lane = threadIdx.x & 31;
  const int gp = lane / NCH, ch = lane % NCH;
  const int npair = (ng + 1) / 2;
  const int g1 = gp, g2 = ng - 1 - gp;
  const int c01 = T + 8 * g1, c02 = T + 8 * g2;
  int64_t a1[8], a2[8];
#pragma unroll
  for (int r = 0; r < 8; r++) a1[r] = a2[r] = 0;
#pragma unroll 1
  for (int k = 0; k < nprod; k++) {
    const Prod P = desc[k];
    if (gp >= npair || P.ia.y < 0 || P.ib.y < 0) continue;
    const int lo1 = max(P.ia.x, c01 - P.ib.y), hi1 = min(P.ia.y, c01 + 7 - P.ib.x);
    int lo2 = 0, hi2 = -1;
    if (g2 > g1) {
      lo2 = max(P.ia.x, c02 - P.ib.y);
      hi2 = min(P.ia.y, c02 + 7 - P.ib.x);
    }
    // this lane's share of the pair's concatenated p-ranges: [s0, s1)
    const int len1 = hi1 >= lo1 ? hi1 - lo1 + 1 : 0, len2 = hi2 >= lo2 ? hi2 - lo2 + 1 : 0;
    const int tot = len1 + len2;
    const int s0 = (ch * tot) / NCH, s1 = ((ch + 1) * tot) / NCH;
    mac_run(a1, P.A, P.B, c01, lo1 + s0, lo1 + min(s1, len1) - 1);
    mac_run(a2, P.A, P.B, c02, lo2 + max(s0 - len1, 0), lo2 + s1 - len1 - 1);
    if (mc && ch == 0) {
      mc->useful += group_macs(P.ia, P.ib, c01) + (g2 > g1 ? group_macs(P.ia, P.ib, c02) : 0);
      mc->executed += 8ull * tot;
    }
  }
  if (!accumulate)
    for (int c = lane; c < ncp; c += 32) sts64(out + 8 * c, 0);
  __syncwarp();
  // reduce-scatter over the NCH lanes of each pair
  int64_t v[16];
#pragma unroll
  for (int r = 0; r < 8; r++) {
    v[r] = a1[r];
    v[8 + r] = a2[r];
  }
  int base = 0;
#pragma unroll
  for (int s = NCH / 2, n = 16; s >= 1; s >>= 1, n >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
      if (j < n / 2) {
        const int64_t send = up ? v[j] : v[n / 2 + j];
        const int64_t keep = up ? v[n / 2 + j] : v[j];
        v[j] = keep + __shfl_xor_sync(0xffffffffu, send, s);
      }
    }
    if (up) base += n / 2;
  }
  if (gp < npair) {
    constexpr int nf = 16 / NCH;
#pragma unroll
    for (int j = 0; j < nf; j++) {
      const int idx = base + j;
      const int g = idx < 8 ? g1 : g2;
      if (idx >= 8 && g2 <= g1) continue;
      const int rel = 8 * g + (idx & 7);
      if (rel < nout) {
        const uint32_t a = out + 8 * rel;
        sts64(a, accumulate ? lds64(a) + v[j] : v[j]);
      }
    }
  }
  __syncwarp();
}

// Several products per warp: lane l works on product l / LPP (LPP = NP2 * 2
// lanes per product, NP2 = group pairs rounded up to a power of two), on group
// pair gp and one half of the pair's p-range; the two halves of a pair are
// reduced with one shuffle round and the exact columns of product k are
// written to out + k * ostride (bytes). Longer per-lane runs (~len/2 p-steps)
// amortise the setup and reduction that dominate short runs.
template <int NP2>
__device__ __noinline__ void warp_multi(const Prod* desc, int nprod, int T, int ng, uint32_t out, int ostride,
                                        int ncp, int nout, MacCount* mc) {
  constexpr int LPP = 2 * NP2;
  const int lane = threadIdx.x & 31;
  const int k = lane / LPP, gp = (lane % LPP) >> 1, ch = lane & 1;
  const int npair = (ng + 1) / 2;
  const bool act = k < nprod && gp < npair;
  const int g1 = gp, g2 = ng - 1 - gp;
  const int c01 = T + 8 * g1, c02 = T + 8 * g2;
  int64_t a1[8], a2[8];
#pragma unroll
  for (int r = 0; r < 8; r++) a1[r] = a2[r] = 0;
  const Prod P = desc[k < nprod ? k : 0];
  if (act && P.ia.y >= 0 && P.ib.y >= 0) {
    const int lo1 = max(P.ia.x, c01 - P.ib.y), hi1 = min(P.ia.y, c01 + 7 - P.ib.x);
    int lo2 = 0, hi2 = -1;
    if (g2 > g1) {
      lo2 = max(P.ia.x, c02 - P.ib.y);
      hi2 = min(P.ia.y, c02 + 7 - P.ib.x);
    }
    const int len1 = hi1 >= lo1 ? hi1 - lo1 + 1 : 0, len2 = hi2 >= lo2 ? hi2 - lo2 + 1 : 0;
    const int tot = len1 + len2;
    const int s0 = ch ? tot / 2 : 0, s1 = ch ? tot : tot / 2;
    mac_run(a1, P.A, P.B, c01, lo1 + s0, lo1 + min(s1, len1) - 1);
    mac_run(a2, P.A, P.B, c02, lo2 + max(s0 - len1, 0), lo2 + s1 - len1 - 1);
    if (mc && ch == 0) {
      mc->useful += group_macs(P.ia, P.ib, c01) + (g2 > g1 ? group_macs(P.ia, P.ib, c02) : 0);
      mc->executed += 8ull * tot;
    }
  }
  // zero-fill the rows of this warp's products, then one reduction round
  for (int e = lane; e < nprod * ncp; e += 32) {
    const int kk = e / ncp, c = e - kk * ncp;
    sts64(out + kk * ostride + 8 * c, 0);
  }
  __syncwarp();
  int64_t v[8];
#pragma unroll
  for (int r = 0; r < 8; r++) {
    const int64_t send = ch ? a1[r] : a2[r];
    const int64_t keep = ch ? a2[r] : a1[r];
    v[r] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
  }
  if (act) {
    const int g = ch ? g2 : g1;
    if (!(ch && g2 <= g1)) {
#pragma unroll
      for (int r = 0; r < 8; r++) {
        const int rel = 8 * g + r;
        if (rel < nout) sts64(out + k * ostride + 8 * rel, v[r]);
      }
    }
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Branch-free lead products. For a product shape (truncation T, full-width
// operands of W and Wb digits) the p-range of every 8-column group g is fixed:
// [max(0, c0 - Wb + 1), min(W - 1, c0 + 7)], c0 = T + 8g. The 32 lanes of a
// warp are dealt to the groups in proportion to their lengths, each lane
// getting one run of <= kRun p-steps of one group (a table computed once per
// kernel). A product is then: 8 + 7 + kRun loads, 8 x kRun IMAD.WIDE with
// compile-time register indices, 8 partial columns to the warp's scratch,
// and a segment sum per column. Zero digits beyond the operands' nonzero
// ranges cost MACs but no branches.
constexpr int kRun = 10;

struct LaneRun {
  int g, p0, ns;  // group, first p, steps (0 = idle)
};

__host__ __device__ inline int grp_len(int g, int T, int W, int Wb) {
  const int c0 = T + 8 * g;
  const int lo = c0 - Wb + 1 > 0 ? c0 - Wb + 1 : 0;
  const int hi = c0 + 7 < W - 1 ? c0 + 7 : W - 1;
  return hi >= lo ? hi - lo + 1 : 0;
}

// lanes per group (sum 32) for a shape; returns the largest run, or -1 if > kRun
__device__ inline int plan_lanes(int T, int W, int Wb, int ng, int* nl) {
  int tot = 0;
  for (int g = 0; g < ng; g++) tot += grp_len(g, T, W, Wb);
  int used = 0;
  for (int g = 0; g < ng; g++) {
    const int len = grp_len(g, T, W, Wb);
    nl[g] = len > 0 ? max(1, (32 * len) / (tot > 0 ? tot : 1)) : 0;
    used += nl[g];
  }
  while (used > 32) {  // take lanes from the group with the shortest resulting runs
    int best = -1, bl = 1 << 30;
    for (int g = 0; g < ng; g++)
      if (nl[g] > 1) {
        const int len = grp_len(g, T, W, Wb), r = (len + nl[g] - 2) / (nl[g] - 1);
        if (r < bl) {
          bl = r;
          best = g;
        }
      }
    if (best < 0) return -1;
    nl[best]--;
    used--;
  }
  while (used < 32) {  // give spare lanes to the group with the longest runs
    int best = -1, bl = -1;
    for (int g = 0; g < ng; g++) {
      const int len = grp_len(g, T, W, Wb);
      if (nl[g] == 0) continue;
      const int r = (len + nl[g] - 1) / nl[g];
      if (r > bl) {
        bl = r;
        best = g;
      }
    }
    if (best < 0) break;
    nl[best]++;
    used++;
  }
  int mx = 0;
  for (int g = 0; g < ng; g++)
    if (nl[g]) mx = max(mx, (grp_len(g, T, W, Wb) + nl[g] - 1) / nl[g]);
  return mx <= kRun ? mx : -1;
}

// this lane's run and the lane range of every group (gl[g] = first lane, gl[ng] = 32)
__device__ inline LaneRun lane_run(int T, int W, int Wb, int ng, int lane, int* gl) {
  int nl[32];
  LaneRun lr{0, 0, 0};
  if (plan_lanes(T, W, Wb, ng, nl) < 0) return lr;
  int first = 0;
  for (int g = 0; g < ng; g++) {
    gl[g] = first;
    const int len = grp_len(g, T, W, Wb);
    if (lane >= first && lane < first + nl[g]) {
      const int k = lane - first;
      const int c0 = T + 8 * g;
      const int lo = c0 - Wb + 1 > 0 ? c0 - Wb + 1 : 0;
      const int s0 = (k * len) / nl[g], s1 = ((k + 1) * len) / nl[g];
      lr = LaneRun{g, lo + s0, s1 - s0};
    }
    first += nl[g];
  }
  gl[ng] = first;
  return lr;
}

// Zero-skipping: the schedule of a product whose operands' top nonzero digits
// are a1, b1 is the one of the shape (T, Wa, Wb) with Wa, Wb the widths
// rounded up to multiples of kQ (digits above a row's top are zero, so the
// result is unchanged). Tables for every (truncation, Wa, Wb) are built once
// per kernel in shared memory: run[shape][lane] and gl[shape][33].

__host__ __device__ inline int shape_id(int tsel, int qa, int qb) { return (tsel * kMaxQ + qa - 1) * kMaxQ + qb - 1; }

// top nonzero digit of a row (warp-wide; -1 if zero)
__device__ __forceinline__ int row_top(const int32_t* A, int W) {
  int t = -1;
  for (int base = 0; base < W; base += 32) {
    const int d = base + (threadIdx.x & 31);
    const unsigned m = __ballot_sync(0xffffffffu, d < W && A[d] != 0);
    if (m) t = base + 31 - __clz(m);
  }
  return t;
}

// this lane's share of A (x) B accumulated into acc (fixed schedule `lr`)
__device__ __forceinline__ void run_acc(int64_t (&acc)[8], const int32_t* A, const int32_t* B, int T, LaneRun lr) {
  {
    const int c0 = T + 8 * lr.g;
    int32_t a[kRun], b[kRun + 7];
#pragma unroll
    for (int u = 0; u < kRun; u++) a[u] = u < lr.ns ? A[lr.p0 + u] : 0;
#pragma unroll
    for (int t = 0; t < kRun + 7; t++) b[t] = B[c0 - lr.p0 - (kRun - 1) + t];  // b[t] = B[c0 - p0 - kRun + 1 + t]
#pragma unroll
    for (int u = 0; u < kRun; u++)
#pragma unroll
      for (int r = 0; r < 8; r++) acc[r] = madw(a[u], b[r - u + kRun - 1], acc[r]);
  }
}

// useful (nonzero-range) digit products of this lane's run: for counters only
__device__ __forceinline__ unsigned long long run_useful(LaneRun lr, int T, int2 ia, int2 ib) {
  if (lr.ns <= 0 || ia.y < 0 || ib.y < 0) return 0;
  const int c0 = T + 8 * lr.g;
  unsigned long long n = 0;
  for (int r = 0; r < 8; r++) {
    const int c = c0 + r;
    const int lo = max(max(ia.x, c - ib.y), lr.p0), hi = min(min(ia.y, c - ib.x), lr.p0 + lr.ns - 1);
    if (hi >= lo) n += hi - lo + 1;
  }
  return n;
}

// the lanes' windows -> exact columns out[0..ncp) (segment sum per group; `gl` = lane table)
__device__ __forceinline__ void run_reduce(const int64_t (&acc)[8], const int* gl, int ng, int64_t* scr, int64_t* out,
                                           int nout, int ncp, bool accumulate = false) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < 8; r++) scr[r * kScrStride + lane] = acc[r];  // column-major, odd stride: no bank conflicts
  __syncwarp();
  for (int c = lane; c < ncp; c += 32) {
    int64_t s = 0;
    if (c < nout && c < 8 * ng) {
      const int g = c >> 3, r = c & 7;
      for (int l = gl[g]; l < gl[g + 1]; l++) s += scr[r * kScrStride + l];
    }
    out[c] = accumulate ? out[c] + s : s;
  }
  __syncwarp();
}

// shape tables (shared): run[shape * 32 + lane] = (group, p0, steps, ok), gl[shape * 33 + g]
__device__ inline void build_shapes(int T, int Tc, int W, int KW, int ng, int4* run, int* gl) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int sh = warp; sh < kShapes; sh += kThreads / 32) {
    const int tsel = sh / (kMaxQ * kMaxQ), qa = (sh / kMaxQ) % kMaxQ + 1, qb = sh % kMaxQ + 1;
    const int Tt = tsel ? Tc : T;
    const int Wa = min(qa * kQ, W), Wb = min(qb * kQ, KW);
    const int ngs = max(0, min(ng, (Wa + Wb - 2 - Tt) / 8 + 1));
    int glt[33];
    int nl[32];
    const bool ok = ngs > 0 && plan_lanes(Tt, Wa, Wb, ngs, nl) >= 0;
    LaneRun lr{0, 0, 0};
    if (ok) lr = lane_run(Tt, Wa, Wb, ngs, lane, glt);
    run[sh * 32 + lane] = make_int4(lr.g, lr.p0, lr.ns, ok ? ngs : 0);
    if (lane == 0 && ok)
      for (int g = 0; g <= ngs; g++) gl[sh * 33 + g] = glt[g];
  }
}

// zero-skipping exact product on one warp: out (=|+=) A (x) B, truncation Tt (tsel),
// A of Wa_full digits, B of Wb_full; falls back to the full-width schedule `lrf`/`glf`
__device__ __forceinline__ void zs_product(const int32_t* A, int Wa_full, const int32_t* B, int Wb_full, int tsel,
                                           int Tt, const int4* run, const int* glbase, LaneRun lrf, const int* glf,
                                           int ngf, int64_t* scr, int64_t* out, int nout, int ncp, bool accumulate,
                                           MacCount* mc) {
  const int lane = threadIdx.x & 31;
  const int a1 = row_top(A, Wa_full), b1 = row_top(B, Wb_full);
  if (a1 < 0 || b1 < 0 || a1 + b1 < Tt) {
    if (!accumulate)
      for (int c = lane; c < ncp; c += 32) out[c] = 0;
    __syncwarp();
    return;
  }
  const int qa = min(a1 / kQ + 1, kMaxQ), qb = min(b1 / kQ + 1, kMaxQ);
  const int sh = shape_id(tsel, qa, qb);
  const int4 rr = run[sh * 32 + lane];
  const bool ok = __shfl_sync(0xffffffffu, rr.w, 0) > 0;
  const LaneRun lr = ok ? LaneRun{rr.x, rr.y, rr.z} : lrf;
  const int* gl = ok ? glbase + sh * 33 : glf;
  const int ng = ok ? rr.w : ngf;
  int64_t acc[8];
#pragma unroll
  for (int r = 0; r < 8; r++) acc[r] = 0;
  run_acc(acc, A, B, Tt, lr);
  run_reduce(acc, gl, ng, scr, out, nout, ncp, accumulate);
  if (mc) mc->executed += 8ull * lr.ns;
}

// exact columns of A (x) B (W- and Wb-digit rows, zero-padded) into out[0..nout):
// `scr` = this warp's scratch (32 x 8 int64), `gl` = the shape's lane table
__device__ __forceinline__ void lead_product(const int32_t* A, const int32_t* B, int T, LaneRun lr, const int* gl,
                                             int ng, int64_t* scr, int64_t* out, int nout, int ncp) {
  int64_t acc[8];
#pragma unroll
  for (int r = 0; r < 8; r++) acc[r] = 0;
  run_acc(acc, A, B, T, lr);
  run_reduce(acc, gl, ng, scr, out, nout, ncp);
}

__device__ __forceinline__ Prod mkprod(const int32_t* A, int2 ia, const int32_t* B, int2 ib) {
  return Prod{smem_u32(A), smem_u32(B), ia, ib};
}

// one product, columns overwritten; `slot` = this warp's descriptor slot (shared)
template <int NCH>
__device__ __forceinline__ void warp_product(Prod* slot, const int32_t* A, int2 ia, const int32_t* B, int2 ib, int T,
                                             const Geo& g, int64_t* out, MacCount* mc) {
  if ((threadIdx.x & 31) == 0) slot[0] = mkprod(A, ia, B, ib);
  __syncwarp();
  warp_prods<NCH>(slot, 1, T, g.ng, smem_u32(out), g.ncp, g.ncols, 0, mc);
}

__device__ __forceinline__ int2 row_info(const int32_t* r, int n) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  int bot = 1 << 30, tp = -1;
  for (int d = lane; d < n; d += 32)
    if (r[d]) {
      bot = min(bot, d);
      tp = max(tp, d);
    }
  bot = __reduce_min_sync(full, bot);
  tp = __reduce_max_sync(full, tp);
  return make_int2(tp >= 0 ? bot : n, tp);
}

// ---------------------------------------------------------------------------
template <int NPT, int NCH, int MS, int MK>
__global__ void __launch_bounds__(kThreads, 1) taylor_mx_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(8) uint64_t s_bar[4];
  __shared__ int s_flag;
  __shared__ int s_em[kMaxD * kMaxD], s_ej[kMaxD * kMaxD], s_dyn[kMaxD * kMaxD];
  __shared__ int s_base[kMaxD], s_full[kMaxD];
  __shared__ Prod s_prod[kWarps][kPerWarpPass];
  __shared__ int4 s_pl[4][kMaxProd];        // lead product lists: (kind, index, side, multiplier)
  __shared__ int s_tr[4][2 * kMaxD + 1];    // per target: first product of the list
  __shared__ int s_gl[3][33];               // lead: first lane of every group, per product shape
  int2* s_cinfo = nullptr;                  // lead: nonzero range of C_i, every order
  __shared__ int s_wq[kWarps];
  cg::cluster_group cluster = cg::this_cluster();
  const int G = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int traj = blockIdx.x / G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Geo g = make_geo(p);
  const Layout L = make_layout(p, G);
  const int Gb = L.Gb;
  const int nE = L.nE;
  const int NPp = p.NP > 0 ? p.NP : 1;
  const int N = p.N;
  MacCount mcount;
  MacCount* mc = p.counters ? &mcount : nullptr;
  int32_t* ktab = (int32_t*)p.gscratch + (size_t)traj * N * nE * g.krs;
  int2* kinfo = (int2*)((int32_t*)p.gscratch + (size_t)p.n_traj * N * nE * g.krs) + (size_t)traj * N * nE;
  int32_t* gstate = p.state + (size_t)traj * p.D * p.RS;

  for (size_t w = tid; w < L.total / 4; w += kThreads) ((int32_t*)smem)[w] = 0;
  if (tid == 0) {
    n_entries(p, s_em, s_ej, s_dyn);
    s_flag = 0;
    for (int b = 0; b < 4; b++) mbar_init(&s_bar[b], 1);
  }
  if (tid < kMaxD) {
    int f = 1;
    s_base[tid] = tid < p.D ? row_slots(p, G, tid, &f) : 0;
    s_full[tid] = f;
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int R_ST = 0, R_SB = p.D, R_LIN = 2 * p.D, R_U = R_LIN + p.D * p.D, R_K = R_U + 2 * p.D,
            R_C = R_K + 2 * nE, R_ROW = R_C + 2, R_ROW1 = R_ROW + 2 * p.D;
  if (rank == 0) {
    int32_t* lrow = (int32_t*)(smem + L.off_lrow) + 2 * kPad;
    for (int r = 0; r < p.D * p.D; r++)
      for (int d = tid; d < p.W; d += kThreads) lrow[(size_t)(R_LIN + r) * g.rs + d] = p.lin[(size_t)r * p.RS + d];
    for (int m = 0; m < p.D; m++)
      for (int d = tid; d < p.W; d += kThreads) lrow[(size_t)(R_ST + m) * g.rs + d] = gstate[(size_t)m * p.RS + d];
  }
  __syncthreads();
  cluster.sync();

  const uint32_t row_bytes = (uint32_t)(g.urs * 4);  // one row (bulk copy)
  const uint32_t recv_bytes = (uint32_t)(Gb * NPp * g.ncp * 8);
  const uint32_t bar_local = smem_u32(&s_bar[0]);
  auto owner = [&](int k) { return 1 + (k - 1) % Gb; };
  auto SLOT = [&](int v, int k) { return s_base[v] + (s_full[v] ? k : k / Gb); };

  if (rank == 0) {
    // =============================== lead ===============================
    int32_t* lrow = (int32_t*)(smem + L.off_lrow) + 2 * kPad;
    int2* linfo = (int2*)(smem + L.off_linfo);
    int64_t* cpart = (int64_t*)(smem + L.off_cpart);
    int64_t* lsum = (int64_t*)(smem + L.off_lsum);
    int64_t* cbuf = (int64_t*)(smem + L.off_cbuf);
    int64_t* recv = (int64_t*)(smem + L.off_recv);
    int64_t* ssum = (int64_t*)(smem + L.off_ssum);
    auto LR = [&](int r) { return lrow + (size_t)r * g.rs; };
    const uint32_t rows_remote = smem_u32(smem + L.off_rows) + 4 * 2 * kPad;
    for (int r = warp; r < R_U; r += kWarps) {
      if (r >= R_SB && r < R_LIN) continue;
      const int2 inf = row_info(LR(r), p.W);
      if (lane == 0) linfo[r] = inf;
    }
    // product lists per order kind (0: j = 1, 1: j = 2, 2: 3 <= j <= N-1, 3: last order, rows only),
    // grouped by target (U_j^0..D-1, then rows 0..D-1), and the C_i nonzero ranges
    if (tid == 0) {
      for (int lk = 0; lk < 4; lk++) {
        const bool doU = lk != 3;
        const int lagn = lk < 3 ? lk : 0;
        int cnt = 0;
        for (int tg = 0; tg < 2 * p.D; tg++) {
          s_tr[lk][tg] = cnt;
          if (tg < p.D && doU) {
            for (int e = 0; e < nE; e++)
              if (s_em[e] == tg) s_pl[lk][cnt++] = make_int4(0, e, 0, 1);
            for (int t = 0; t < p.NT; t++)
              if (p.teq[t] == tg)
                for (int side = 0; side < lagn; side++) s_pl[lk][cnt++] = make_int4(2, t, side, p.tq_int[t]);
          } else if (tg >= p.D) {
            s_pl[lk][cnt++] = make_int4(1, tg - p.D, 0, 1);
          }
        }
        s_tr[lk][2 * p.D] = cnt;
      }
    }
    // branch-free product schedules: shapes 0 = U x K (Tc, W, W+1), 1 = U x C (Tc, W, W), 2 = row x row (T, W, W)
    const LaneRun lr0 = lane_run(g.Tc, p.W, g.KW, g.ng, lane, s_gl[0]);
    const LaneRun lr1 = lane_run(g.Tc, p.W, p.W, g.ng, lane, s_gl[1]);
    const LaneRun lr2 = lane_run(g.T, p.W, p.W, g.ng, lane, s_gl[2]);
    int nlt[32];
    const bool fast = g.ng <= 32 && plan_lanes(g.Tc, p.W, g.KW, g.ng, nlt) >= 0 &&
                      plan_lanes(g.Tc, p.W, p.W, g.ng, nlt) >= 0 && plan_lanes(g.T, p.W, p.W, g.ng, nlt) >= 0;
    int64_t* scr = (int64_t*)(smem + L.off_scr) + (size_t)warp * kScrStride * 8;
    int4* shr = (int4*)(smem + L.off_lshr);
    int* shg = (int*)(smem + L.off_lshg);
    // zero-skipping schedules (zs_product) measured slower at K=500: the per-product
    // segment reduction costs more than the skipped MACs; off until the reduction is fused
    constexpr bool zskip = false;
    if (zskip) build_shapes(g.T, g.Tc, p.W, g.KW, g.ng, shr, shg);
    s_cinfo = (int2*)(smem + L.off_cinf);
    for (int i = warp; i < N; i += kWarps) {
      int bot = 1 << 30, tp = -1;
      for (int d = lane; d < p.W; d += 32)
        if (p.ctab[(size_t)i * p.RS + d]) {
          bot = min(bot, d);
          tp = max(tp, d);
        }
      bot = __reduce_min_sync(0xffffffffu, bot);
      tp = __reduce_max_sync(0xffffffffu, tp);
      if (lane == 0) s_cinfo[i] = make_int2(tp >= 0 ? bot : p.W, tp);
    }
    __syncthreads();
    uint32_t rph = 0;

    // warp-wide: publish new row m (index r) through the global coefficient table:
    // one TMA multicast into every bulk CTA for left-hand variables, one copy to
    // the owner of r otherwise
    int32_t* gcoef = p.coef + (size_t)traj * p.D * (N + 1) * p.RS;
    auto push_row = [&](int m, int r, const int32_t* src) {
      int32_t* gdst = gcoef + ((size_t)m * (N + 1) + r) * p.RS;
      for (int d = lane; d < p.RS; d += 32) gdst[d] = d < p.W ? src[d] : 0;
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        const int sl = SLOT(m, r);
        const uint32_t rb_local = bar_local + 8 * (r & 3);
        if (r == 2 && !s_full[m]) {  // row 2 of every variable is kept by every bulk CTA
          const int s2 = L.nslots - p.D + m;
          bulk_multicast(rows_remote + 4 * s2 * g.rs, gdst, (uint32_t)(g.urs * 4), rb_local,
                         (uint16_t)(((1u << G) - 1u) & ~1u));
        }
        if (s_full[m]) {
          bulk_multicast(rows_remote + 4 * sl * g.rs, gdst, (uint32_t)(g.urs * 4), rb_local,
                         (uint16_t)(((1u << G) - 1u) & ~1u));
        } else {
          const int dst = owner(r);
          bulk_push(mapa_u32(rows_remote + 4 * sl * g.rs, dst), smem_u32(src), (uint32_t)(g.urs * 4),
                    mapa_u32(rb_local, dst));
          bulk_commit();
        }
      }
    };
    // C_i into buffer b (cp.async, 16-byte chunks; ctab rows are RS-strided, RS >= W, multiple of 4)
    auto prefetch_c = [&](int i, int b) {
      if (warp == kWarps - 1) {
        const int32_t* src = p.ctab + (size_t)i * p.RS;
        int32_t* dst = LR(R_C + b);
        for (int c = lane; c < p.RS / 4; c += 32)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + 4 * c)), "l"(src + 4 * c)
                       : "memory");
      }
    };
    auto prefetch_k = [&](int i, int b) {
      for (int e = warp; e < nE; e += kWarps) {
        const int32_t* src = ktab + ((size_t)i * nE + e) * g.krs;
        int32_t* dst = LR(R_K + b * nE + e);
        for (int c = lane; c < g.krs / 4; c += 32)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + 4 * c)), "l"(src + 4 * c)
                       : "memory");
        if (lane == 0) linfo[R_K + b * nE + e] = __ldcg(kinfo + (size_t)i * nE + e);
      }
    };

    for (int n = p.start_step + 1; n <= p.n_steps; n++) {
      // ---- step start: row 0 = state (ssum), SB = bnf(state), U_0
      for (int m = 0; m < p.D; m++)
        for (int d = tid; d < p.W + 3; d += kThreads) ssum[(size_t)m * (p.W + 3) + d] = d < p.W ? LR(R_ST + m)[d] : 0;
      if (p.write_coef)
        for (int m = 0; m < p.D; m++)
          for (int d = tid; d < p.W; d += kThreads)
            p.coef[(((size_t)traj * p.D + m) * (N + 1)) * p.RS + d] = LR(R_ST + m)[d];
      if (warp < p.D) {  // SB_m = bnf(state_m)
        int64_t* cv = cbuf + (size_t)warp * g.ncp;
        for (int c = lane; c < g.ncp; c += 32) cv[c] = c == 0 ? -(kRadix / 2) : (c >= 2 && c - 2 < p.W ? LR(R_ST + warp)[c - 2] : 0);
        __syncwarp();
        if (warp_bnf<MS>(cv, g.ncols, p.W, LR(R_SB + warp), &linfo[R_SB + warp]) && lane == 0) atomicOr(&s_flag, 1);
      }
      __syncthreads();
      {
        // products: lin[m][j] (x) SB_j, q_t SB_a (x) SB_b
        int np = 0;
        for (int m = 0; m < p.D; m++)
          for (int j = 0; j < p.D; j++) {
            const int r = R_LIN + m * p.D + j;
            if (linfo[r].y < 0) continue;
            if (np % kWarps == warp)
              warp_product<NCH>(s_prod[warp], LR(r), linfo[r], LR(R_SB + j), linfo[R_SB + j], g.T, g, cpart + (size_t)np * g.ncp, mc);
            np++;
          }
        for (int t = 0; t < p.NT; t++) {
          const int a = p.pj[p.tpair[t]], b = p.pk[p.tpair[t]];
          if (np % kWarps == warp)
            warp_product<NCH>(s_prod[warp], LR(R_SB + a), linfo[R_SB + a], LR(R_SB + b), linfo[R_SB + b], g.T, g,
                              cpart + (size_t)np * g.ncp, mc);
          np++;
        }
        __syncthreads();
        if (warp < p.D) {
          const int m = warp;
          int64_t* cv = cbuf + (size_t)m * g.ncp;
          for (int c = lane; c < g.ncols; c += 32) {
            int64_t s = 0;
            int k = 0;
            for (int mm = 0; mm < p.D; mm++)
              for (int j = 0; j < p.D; j++) {
                if (linfo[R_LIN + mm * p.D + j].y < 0) continue;
                if (mm == m) s += cpart[(size_t)k * g.ncp + c];
                k++;
              }
            for (int t = 0; t < p.NT; t++, k++)
              if (p.teq[t] == m) s += (int64_t)p.tq_int[t] * cpart[(size_t)k * g.ncp + c];
            if (c >= 2 && c - 2 < p.W) s += p.cst[(size_t)m * p.RS + c - 2];
            cv[c] = s;
          }
          __syncwarp();
          if (warp_snf_call<MS>(cv, g.ncols, p.W, LR(R_U + m), &linfo[R_U + m]) && lane == 0) atomicOr(&s_flag, 1);
        }
      }
      prefetch_c(0, 0);
      asm volatile("cp.async.commit_group;" ::: "memory");
      __syncthreads();
      cluster_barrier();  // [C] the K table of this step is complete
      if (N >= 2) prefetch_k(0, 0);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();

      // column-sum pass: this thread's first item (target, column) and the bilinear terms of a
      // U target are the same for every order -- out of the loop (runtime-indexed constant-bank
      // loads and the division cost the single-issue critical path ~1 K cycles per order)
      const int cs_ntg = 2 * p.D;
      const bool cs_on = tid < cs_ntg * g.ncols;
      const int cs_tg = cs_on ? tid / g.ncols : 0, cs_c = cs_on ? tid - cs_tg * g.ncols : 0;
      int cs_nt = 0, cs_q[4] = {0, 0, 0, 0}, cs_coef[4] = {0, 0, 0, 0};
      bool cs_many = false;  // more than four terms in one equation: the generic loop
      if (cs_on && cs_tg < p.D)
        for (int t = 0; t < p.NT; t++)
          if (p.teq[t] == cs_tg) {
            if (cs_nt < 4) {
              cs_q[cs_nt] = p.tpair[t];
              cs_coef[cs_nt] = p.tq_int[t];
              cs_nt++;
            } else {
              cs_many = true;
            }
          }
      cs_many = __syncthreads_or(cs_many) != 0;
      int ssum_lag = 0;  // rows of the previous order still to be added to the state sum (aux warp)

      for (int i = 0; i < N; i++) {
        const int par = i & 1, j = i + 1;
        const bool tlog = p.dbg && n == p.start_step + 1 && i < 256 && lane == 0;
#define LT(k) \
  if (tlog) p.dbg[((size_t)i * 16 + warp) * 8 + (k)] = (long long)clock64();
        LT(0);
        const bool doU = j <= N - 1;
        const int lagn = (j >= 2 && j <= N - 1) ? (j == 2 ? 1 : 2) : 0;
        const int lk = !doU ? 3 : lagn;  // product list of this order
        const int P = s_tr[lk][2 * p.D];
        // prefetch C_{i+1}, K_{i+1} (their buffers were last read at order i-1)
        if (i + 1 < N) prefetch_c(i + 1, par ^ 1);
        if (i + 2 < N) prefetch_k(i + 1, par ^ 1);
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (warp < kMacWarps) {
#pragma unroll 1
          for (int pi = warp; pi < P; pi += kMacWarps) {
            const int4 d = s_pl[lk][pi];  // kind, index, side, -
            const int32_t *A, *B;
            int2 ia, ib;
            int T = g.Tc;
            if (d.x == 0) {  // K entry
              const int e = d.y, ru = R_U + par * p.D + s_ej[e];
              A = LR(ru);
              ia = linfo[ru];
              B = LR(R_K + par * nE + e);
              ib = linfo[R_K + par * nE + e];
            } else if (d.x == 1) {  // new row
              const int ru = R_U + par * p.D + d.y;
              A = LR(ru);
              ia = linfo[ru];
              B = LR(R_C + par);
              ib = s_cinfo[i];
            } else {  // lag-1 term of bilinear term t = d.y (rows j-1 and 1)
              const int t = d.y, a = p.pj[p.tpair[t]], b = p.pk[p.tpair[t]];
              const int ra = (lagn == 2 && d.z == 1) ? R_ROW1 + a : R_ROW + par * p.D + a;
              const int rb = (lagn == 2 && d.z == 0) ? R_ROW1 + b : R_ROW + par * p.D + b;
              A = LR(ra);
              ia = linfo[ra];
              B = LR(rb);
              ib = linfo[rb];
              T = g.T;
            }
            if (zskip) {
              const LaneRun lr = d.x == 0 ? lr0 : (d.x == 1 ? lr1 : lr2);
              zs_product(A, p.W, B, d.x == 0 ? g.KW : p.W, d.x == 2 ? 0 : 1, T, shr, shg, lr, s_gl[d.x], g.ng, scr,
                         cpart + (size_t)pi * g.ncp, g.ncols, g.ncp, false, mc);
            } else if (fast) {
              const LaneRun lr = d.x == 0 ? lr0 : (d.x == 1 ? lr1 : lr2);
              lead_product(A, B, T, lr, s_gl[d.x], g.ng, scr, cpart + (size_t)pi * g.ncp, g.ncols, g.ncp);
              if (mc) {
                mcount.useful += run_useful(lr, T, ia, ib);
                mcount.executed += 8ull * kRun;
              }
            } else {
              warp_product<NCH>(s_prod[warp], A, ia, B, ib, T, g, cpart + (size_t)pi * g.ncp, mc);
            }
          }
        } else {
          // aux warp: the rows rounded at the previous order join the state sum here, off the
          // row warps' critical path (their buffer is rewritten two orders later)
          if (ssum_lag) {
            for (int m = 0; m < p.D; m++) {
              const int32_t* rw = LR(R_ROW + par * p.D + m);
              for (int d = lane; d < p.W; d += 32) ssum[(size_t)m * (p.W + 3) + d] += rw[d];
            }
          }
          // wait for the bulk CTAs' L'(j) (gathered in the column-sum pass below)
          const bool have = doU && j >= 4 && p.NP > 0;
          if (have) {
            const int rp = j & 1;
            if (lane == 0) mbar_expect(&s_bar[rp], recv_bytes);
            mbar_wait(&s_bar[rp], (rph >> rp) & 1);
            rph ^= 1u << rp;
          }
        }
        LT(1);
        __syncthreads();
        LT(2);
        // ---- column sums of every target on all warps, then the roundings:
        //      U_j^m (warps 0..D-1), rows a~_{i+1}^m (warps D..2D-1)
        {
          const int ntg = cs_ntg;
          for (int e = tid; e < ntg * g.ncols; e += kThreads) {
            const bool firstitem = e == tid;
            const int tg = firstitem ? cs_tg : e / g.ncols, c = firstitem ? cs_c : e - tg * g.ncols;
            const bool isU = tg < p.D;
            if (isU && !doU) continue;
            const int k0 = s_tr[lk][tg], k1 = s_tr[lk][tg + 1];
            int64_t sacc = 0;
            if (isU && doU && j >= 4 && p.NP > 0) {  // q_t * sum over the bulk CTAs of L'_t(j)
              const int64_t* rv = recv + (size_t)(j & 1) * Gb * NPp * g.ncp;
              if (firstitem && !cs_many) {
#pragma unroll
                for (int tt = 0; tt < 4; tt++) {
                  if (tt < cs_nt) {
                    const int64_t* rq = rv + (size_t)cs_q[tt] * g.ncp + c;
                    int64_t v = 0;
#pragma unroll 5
                    for (int r = 0; r < Gb; r++) v += rq[(size_t)r * NPp * g.ncp];
                    sacc += (int64_t)cs_coef[tt] * v;
                  }
                }
              } else {
                for (int t = 0; t < p.NT; t++) {
                  if (p.teq[t] != tg) continue;
                  const int q = p.tpair[t];
                  int64_t v = 0;
#pragma unroll 5
                  for (int r = 0; r < Gb; r++) v += rv[((size_t)r * NPp + q) * g.ncp + c];
                  sacc += (int64_t)p.tq_int[t] * v;
                }
              }
            }
            for (int k = k0; k < k1; k++) sacc += (int64_t)s_pl[lk][k].w * cpart[(size_t)k * g.ncp + c];
            cbuf[(size_t)tg * g.ncp + c] = sacc;
          }
        }
        __syncthreads();
        if (warp < 2 * p.D) {
          const int tg = warp;
          const bool isU = tg < p.D;
          const int m = isU ? tg : tg - p.D;
          if (!isU || doU) {
            int64_t* cv = cbuf + (size_t)tg * g.ncp;
            const int rr = isU ? R_U + (par ^ 1) * p.D + m : R_ROW + (par ^ 1) * p.D + m;
            if (!isU && lane == 0) bulk_wait_read();  // the owner copy of row i-1 (same buffer) has read it
            __syncwarp();
            if (warp_snf_call<MS>(cv, g.ncols, p.W, LR(rr), &linfo[rr]) && lane == 0) atomicOr(&s_flag, 1);
            if (!isU) {  // row a~_j: publish, state sum, keep row 1
              __syncwarp();
              push_row(m, j, LR(rr));
              if (i == 0) {
                for (int d = lane; d < p.W; d += 32) LR(R_ROW1 + m)[d] = LR(rr)[d];
                if (lane == 0) linfo[R_ROW1 + m] = linfo[rr];
              }
            }
          }
        }
        LT(3);
        asm volatile("cp.async.wait_all;" ::: "memory");
        LT(4);
        __syncthreads();
        LT(5);
        ssum_lag = 1;
#undef LT
      }
      // the rows of the last order (buffer (N & 1))
      if (warp == kWarps - 1 && N > 0) {
        for (int m = 0; m < p.D; m++) {
          const int32_t* rw = LR(R_ROW + (N & 1) * p.D + m);
          for (int d = lane; d < p.W; d += 32) ssum[(size_t)m * (p.W + 3) + d] += rw[d];
        }
      }
      if (lane == 0) bulk_wait_read();
      __syncthreads();
      // ---- end of step: state = RN_P(sum of rows)
      if (warp < p.D) {
        const int m = warp;
        if (warp_canon(ssum + (size_t)m * (p.W + 3), p.W + 3, p.W, LR(R_ST + m), &linfo[R_ST + m], p.P) && lane == 0)
          atomicOr(&s_flag, 1);
        if ((n % p.stride == 0) || (n == p.n_steps)) {
          const int slot = (n % p.stride == 0) ? (n / p.stride - p.start_step / p.stride)
                                               : (p.n_steps / p.stride - p.start_step / p.stride + 1);
          int32_t* dst = p.rec + ((size_t)slot * p.n_traj + traj) * p.D * p.RS + (size_t)m * p.RS;
          for (int d = lane; d < p.W; d += 32) dst[d] = LR(R_ST + m)[d];
        }
      }
      __syncthreads();
      cluster_barrier();  // [B] the new state is visible to the bulk CTAs
    }
    for (int m = 0; m < p.D; m++)
      for (int d = tid; d < p.W; d += kThreads) gstate[(size_t)m * p.RS + d] = LR(R_ST + m)[d];
  } else {
    // =============================== bulk ===============================
    const int o = rank;
    int32_t* rows = (int32_t*)(smem + L.off_rows) + 2 * kPad;
    int2* rinfo = (int2*)(smem + L.off_rinfo);
    int32_t* srow = (int32_t*)(smem + L.off_srow) + kPad;
    int2* sinfo = (int2*)(smem + L.off_sinfo);
    int32_t* crow = (int32_t*)(smem + L.off_crow) + kPad;
    int2* cinfo = (int2*)(smem + L.off_cinfo);
    int64_t* wcol = (int64_t*)(smem + L.off_wcol);
    int64_t* accA = (int64_t*)(smem + L.off_acc);
    int64_t* accB = (int64_t*)(smem + L.off_bcc);
    int32_t* kst = (int32_t*)(smem + L.off_kst);
    int64_t* kcol = (int64_t*)(smem + L.off_kcol);
    auto ROW = [&](int v, int k) { return rows + (size_t)SLOT(v, k) * g.rs; };
    auto RINF = [&](int v, int k) { return rinfo[SLOT(v, k)]; };
    auto ROW2 = [&](int v) {  // row 2 of variable v (every bulk CTA)
      return s_full[v] ? ROW(v, 2) : rows + (size_t)(L.nslots - p.D + v) * g.rs;
    };
    const uint32_t recv_remote = smem_u32(smem + L.off_recv);
    const int32_t* lead_state = cluster.map_shared_rank((int32_t*)(smem + L.off_lrow) + 2 * kPad, 0);
    uint32_t rph4 = 0;  // phase bits of the 4 row barriers
    // branch-free schedule for row x row products (shape T, W, W)
    const LaneRun lrb = lane_run(g.T, p.W, p.W, g.ng, lane, s_gl[2]);
    int nlb[32];
    const bool bfast = g.ng <= 32 && plan_lanes(g.T, p.W, p.W, g.ng, nlb) >= 0;
    int64_t* bscr = (int64_t*)(smem + L.off_bscr) + (size_t)warp * kScrStride * 8;
    int4* bshr = (int4*)(smem + L.off_bshr);
    int* bshg = (int*)(smem + L.off_bshg);
    constexpr bool bzskip = false;
    if (bzskip) build_shapes(g.T, g.Tc, p.W, g.KW, g.ng, bshr, bshg);
    __syncthreads();
    int nfull = 0;
    for (int v = 0; v < p.D; v++) nfull += s_full[v];

    // exact per-CTA accumulation: every warp's exact partial columns -> (A, B) = (sum of low digits, sum of carries)
    auto absorb = [&](int nw_used) {
      __syncthreads();
      // two columns per thread; the pair list s_wq is read once into registers
      uint32_t wmask[kMaxP] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int w = 0; w < nw_used; w++)
        if (s_wq[w] >= 0) wmask[s_wq[w]] |= 1u << w;
      const int nh = g.ncp / 2;
      for (int e = tid; e < p.NP * nh; e += kThreads) {
        const int q = e / nh, c = 2 * (e - q * nh);
        int64_t a0 = 0, b0 = 0, a1 = 0, b1 = 0;
        uint32_t m = q == 0 ? wmask[0] : q == 1 ? wmask[1] : q == 2 ? wmask[2] : wmask[3];
        while (m) {
          const int w = __ffs(m) - 1;
          m &= m - 1;
          const longlong2 v = *(const longlong2*)(wcol + (size_t)w * g.ncp + c);
          a0 += v.x & kMask;
          b0 += v.x >> kRadixBits;
          a1 += v.y & kMask;
          b1 += v.y >> kRadixBits;
        }
        longlong2* pa = (longlong2*)(accA + (size_t)q * g.ncp + c);
        longlong2* pb = (longlong2*)(accB + (size_t)q * g.ncp + c);
        const longlong2 xa = *pa, xb = *pb;
        *pa = make_longlong2(xa.x + a0, xa.y + a1);
        *pb = make_longlong2(xb.x + b0, xb.y + b1);
      }
      __syncthreads();
    };

    for (int n = p.start_step + 1; n <= p.n_steps; n++) {
      const bool first = n == p.start_step + 1;
      if (tid == 0) bulk_wait_read();  // the last push of the previous step has read the staging area
      __syncthreads();
      // ---- S^e = bnf(lin + q state) (exact)
      for (int e = tid; e < NPp * g.ncp; e += kThreads) accA[e] = accB[e] = 0;
      if (warp < nE) {
        const int e = warp, m = s_em[e], j = s_ej[e];
        int64_t* cv = kcol + (size_t)e * g.ncp;
        for (int c = lane; c < g.ncp; c += 32) {
          int64_t s = 0;
          if (c == 0) s = -(kRadix / 2);
          if (c >= 2 && c - 2 < p.W) {
            const int d = c - 2;
            s = p.lin[(size_t)(m * p.D + j) * p.RS + d];
            for (int t = 0; t < p.NT; t++) {
              if (p.teq[t] != m) continue;
              const int a = p.pj[p.tpair[t]], b = p.pk[p.tpair[t]];
              if (a == j) s += (int64_t)p.tq_int[t] * lead_state[(size_t)b * g.rs + d];
              if (b == j) s += (int64_t)p.tq_int[t] * lead_state[(size_t)a * g.rs + d];
            }
          }
          cv[c] = s;
        }
        __syncwarp();
        if (warp_bnf<MS>(cv, g.ncols, p.W, srow + (size_t)e * g.rs, &sinfo[e]) && lane == 0) atomicOr(&s_flag, 1);
      }
      __syncthreads();
      // ---- K_i^e = rnd_{KW}(S^e (x) C_i), i = o-1, o-1+Gb, ... < N-1; state-free entries only once
      for (int i = o - 1; i + 1 < N; i += Gb) {
        for (int d = tid; d < p.W; d += kThreads) crow[d] = __ldg(p.ctab + (size_t)i * p.RS + d);
        __syncthreads();
        if (warp == 0) {
          const int2 inf = row_info(crow, p.W);
          if (lane == 0) cinfo[0] = inf;
        }
        __syncthreads();
        for (int e = warp; e < nE; e += kWarps) {
          if (!first && !s_dyn[e]) continue;
          int64_t* cv = kcol + (size_t)warp * g.ncp;
          warp_product<NCH>(s_prod[warp], srow + (size_t)e * g.rs, sinfo[e], crow, cinfo[0], g.T, g, cv, mc);
          int2 inf;
          int32_t* out = kst + (size_t)warp * g.krs;
          if (warp_snf_call<MK>(cv, g.ncols, g.KW, out, &inf) && lane == 0) atomicOr(&s_flag, 1);
          __syncwarp();
          int32_t* dst = ktab + ((size_t)i * nE + e) * g.krs;
          for (int d = lane; d < g.krs; d += 32) dst[d] = d < g.KW ? out[d] : 0;
          if (lane == 0) kinfo[(size_t)i * nE + e] = inf;
        }
        __syncthreads();
      }
      cluster_barrier();  // [C]

      for (int r = 1; r <= N; r++) {
        const bool own = owner(r) == o;
        const int rb = r & 3;
        const bool blog = p.dbg && n == p.start_step + 1 && r < 256 && tid == 0 && o <= 2;
#define BT(k) \
  if (blog) p.dbg[40000 + ((size_t)(o - 1) * 256 + r) * 8 + (k)] = (long long)clock64();
        BT(0);
        if (tid == 0)
          mbar_expect(&s_bar[rb], row_bytes * (uint32_t)((own ? p.D : nfull) + (r == 2 ? p.D - nfull : 0)));
        mbar_wait(&s_bar[rb], (rph4 >> rb) & 1);
        rph4 ^= 1u << rb;
        BT(1);
        if (!bfast) {  // nonzero ranges of the rows that arrived (range-aware products only)
          if (warp < p.D && (own || s_full[warp])) {
            const int2 inf = row_info(ROW(warp, r), p.W);
            if (lane == 0) rinfo[SLOT(warp, r)] = inf;
          }
          __syncthreads();
        }
        // (a) new terms of L'(r+2): k = 2 (rows r, 2) in owner(2); k = r (rows 2, r) in owner(r), r != 2
        const bool push = r >= 2 && r + 2 <= N - 1 && p.NP > 0;
        int nw = 0;
        if (push) {
          if (tid == 0) bulk_wait_read();  // the previous push has read the staging buffer
          for (int q = 0; q < p.NP; q++) {
            const int a = p.pj[q], b = p.pk[q];
            for (int side = 0; side < 2; side++) {
              // both new terms (rows r, 2) and (2, r) belong to the newest row's owner
              const bool mine = own && (side == 0 || r != 2);
              if (!mine) continue;
              const int32_t* A = side == 0 ? ROW(a, r) : ROW(a, 2);
              const int32_t* Bq = side == 0 ? ROW2(b) : ROW(b, r);
              if (nw == warp) {
                if (bfast) {
                  lead_product(A, Bq, g.T, lrb, s_gl[2], g.ng, bscr, wcol + (size_t)nw * g.ncp, g.ncols, g.ncp);
                  if (mc) {
                    mcount.useful += run_useful(lrb, g.T, make_int2(0, row_top(A, p.W)), make_int2(0, row_top(Bq, p.W)));
                    mcount.executed += 8ull * kRun;
                  }
                }
                else {
                  const int2 ia = side == 0 ? RINF(a, r) : RINF(a, 2);
                  const int2 ib = side == 0 ? (s_full[b] ? RINF(b, 2) : make_int2(0, p.W - 1)) : RINF(b, r);
                  warp_product<NCH>(s_prod[warp], A, ia, Bq, ib, g.T, g, wcol + (size_t)nw * g.ncp, mc);
                }
              }
              if (tid == 0) s_wq[nw] = q;
              nw++;
            }
          }
          __syncthreads();
          // (b) one pass: P_o = old (accA, accB) + new terms; staging = split1(P_o), two columns per thread
          // (column c-1 of the pair is recomputed from the raw sums, so no second pass is needed)
          int64_t* stg = kcol;
          const int nh = g.ncp / 2;
          for (int e = tid; e < p.NP * nh; e += kThreads) {
            const int q = e / nh, c = 2 * (e - q * nh);
            int64_t A[3], Bc[3];
#pragma unroll
            for (int u = 0; u < 3; u++) {
              const int cc = c - 1 + u;
              int64_t av = 0, bv = 0;
              if (cc >= 0 && cc < g.ncols) {
                av = accA[(size_t)q * g.ncp + cc];
                bv = accB[(size_t)q * g.ncp + cc];
                for (int w = 0; w < nw; w++)
                  if (s_wq[w] == q) {
                    const int64_t v = wcol[(size_t)w * g.ncp + cc];
                    av += v & kMask;
                    bv += v >> kRadixBits;
                  }
              }
              A[u] = av;
              Bc[u] = bv;
            }
            stg[(size_t)q * g.ncp + c] = c < g.ncols ? (A[1] & kMask) + (A[0] >> kRadixBits) + Bc[0] : 0;
            stg[(size_t)q * g.ncp + c + 1] = c + 1 < g.ncols ? (A[2] & kMask) + (A[1] >> kRadixBits) + Bc[1] : 0;
          }
          __syncthreads();
          if (tid == 0) {
            const int j = r + 2;
            fence_async_smem();
            const uint32_t off = (uint32_t)((((size_t)(j & 1) * Gb + (o - 1)) * NPp) * g.ncp * 8);
            bulk_push(mapa_u32(recv_remote + off, 0), smem_u32(stg), (uint32_t)(p.NP * g.ncp * 8),
                      mapa_u32(bar_local + 8 * (j & 1), 0));
            bulk_commit();
          }
        }
        BT(2);
        BT(3);
        // (c) old terms of L'(r+3): k in [3, r] owned, rows r+3-k and k; (accA, accB) are overwritten
        // whenever the next row pushes (even with no owned k)
        if (r + 1 >= 2 && r + 3 <= N - 1 && p.NP > 0) {
          int kfirst = 3 + ((o - 1) - (3 - 1) % Gb + Gb) % Gb;  // smallest k >= 3 with owner(k) == o
          const int nk = (r >= 3 && kfirst <= r) ? (r - kfirst) / Gb + 1 : 0;
          const int wpp = kWarps / p.NP;  // warps per pair: warp w -> pair w % NP, k index w / NP (+ stride)
          if (tid < kWarps) s_wq[tid] = (tid < wpp * p.NP) ? tid % p.NP : -1;
          for (int base = 0; base == 0 || base < nk; base += wpp * kPerWarpPass) {
            if (warp < wpp * p.NP) {
              const int q = warp % p.NP, kw = warp / p.NP;
              const int a = p.pj[q], b = p.pk[q];
              if (bfast) {
                int64_t acc[8];
#pragma unroll
                for (int u = 0; u < 8; u++) acc[u] = 0;
#pragma unroll 1
                for (int u = 0; u < kPerWarpPass; u++) {
                  const int kk = base + kw + u * wpp;
                  if (kk >= nk) break;
                  const int k = kfirst + kk * Gb;
                  run_acc(acc, ROW(a, r + 3 - k), ROW(b, k), g.T, lrb);
                  if (mc) {
                    mcount.useful += run_useful(lrb, g.T, make_int2(0, row_top(ROW(a, r + 3 - k), p.W)),
                                                make_int2(0, row_top(ROW(b, k), p.W)));
                    mcount.executed += 8ull * kRun;
                  }
                }
                run_reduce(acc, s_gl[2], g.ng, bscr, wcol + (size_t)warp * g.ncp, g.ncols, g.ncp);
              } else {
                int np = 0;
                for (int u = 0; u < kPerWarpPass; u++) {
                  const int kk = base + kw + u * wpp;
                  if (kk >= nk) break;
                  const int k = kfirst + kk * Gb;
                  if (lane == 0) s_prod[warp][u] = mkprod(ROW(a, r + 3 - k), RINF(a, r + 3 - k), ROW(b, k), RINF(b, k));
                  np = u + 1;
                }
                __syncwarp();
                warp_prods<NCH>(s_prod[warp], np, g.T, g.ng, smem_u32(wcol + (size_t)warp * g.ncp), g.ncp, g.ncols, 0,
                                mc);
              }
            }
            __syncthreads();
            // (A, B) = sums of the warps' low digits / carries; the first pass overwrites
            const int nh = g.ncp / 2;
            for (int e = tid; e < p.NP * nh; e += kThreads) {
              const int q = e / nh, c = 2 * (e - q * nh);
              int64_t a0 = 0, b0 = 0, a1 = 0, b1 = 0;
              for (int w = q; w < wpp * p.NP; w += p.NP) {
                const longlong2 v = *(const longlong2*)(wcol + (size_t)w * g.ncp + c);
                a0 += v.x & kMask;
                b0 += v.x >> kRadixBits;
                a1 += v.y & kMask;
                b1 += v.y >> kRadixBits;
              }
              longlong2* pa = (longlong2*)(accA + (size_t)q * g.ncp + c);
              longlong2* pb = (longlong2*)(accB + (size_t)q * g.ncp + c);
              if (base == 0) {
                *pa = make_longlong2(a0, a1);
                *pb = make_longlong2(b0, b1);
              } else {
                const longlong2 xa = *pa, xb = *pb;
                *pa = make_longlong2(xa.x + a0, xa.y + a1);
                *pb = make_longlong2(xb.x + b0, xb.y + b1);
              }
            }
            __syncthreads();
          }
        }
        BT(4);
#undef BT
      }
      cluster_barrier();  // [B]
    }
  }
  bulk_wait_read();  // bulk copies issued by this thread have read their sources
  __syncthreads();
  cluster.sync();
  if (rank != 0 && tid == 0 && (s_flag & 1)) {
    int* lead_flag = cluster.map_shared_rank(&s_flag, 0);
    atomicOr(lead_flag, 1);
  }
  cluster.sync();
  if (rank == 0 && tid == 0) p.status[traj] = (s_flag & 1) ? kOverflow : kOk;
  if (mc) {
    atomicAdd(&p.counters[0], mcount.useful);
    atomicAdd(&p.counters[1], mcount.executed);
  }
}

}  // namespace mx

size_t mx_smem_bytes(const Params& p, int G) { return mx::make_layout(p, G).total; }

size_t mx_scratch_bytes(const Params& p) {
  const mx::Geo g = mx::make_geo(p);
  const int nE = mx::n_entries(p, nullptr, nullptr);
  return (size_t)p.n_traj * p.N * nE * (g.krs * 4 + 8);
}

bool mx_supported(const Params& p) {
  const mx::Geo g = mx::make_geo(p);
  int em[kMaxD * kMaxD], ej[kMaxD * kMaxD];
  const int nE = mx::n_entries(p, em, ej);
  // exact int64 column sums on the lead: products per U target x (W 2^54 + 2^56) < 2^63
  int worst = 0;
  for (int m = 0; m < p.D; m++) {
    int c = 0;
    for (int e = 0; e < nE; e++) c += em[e] == m;
    for (int t = 0; t < p.NT; t++) c += 2 * (p.teq[t] == m);
    worst = c > worst ? c : worst;
  }
  const double bound = (double)worst * ((double)p.W * 18014398509481984.0 + 72057594037927936.0);
  const int nlag = 2 * p.NT;
  return p.D <= kMaxD && p.all_q_small && p.NP >= 1 && p.NP <= 4 && nE + p.D + nlag <= mx::kMaxProd &&
         2 * p.D <= mx::kWarps && nE <= mx::kWarps && g.W <= 120 && bound < 9.0e18 &&
         mx::kWarps / p.NP >= 1 && mx::snf_m(g.KW) <= 4;
}

template <int NPT, int NCH>
static const void* mx_fn_ms(int ms, int mk) {
#define MXK(A, B) (const void*)mx::taylor_mx_kernel<NPT, NCH, A, B>
  if (ms == 1) return mk == 1 ? MXK(1, 1) : MXK(1, 2);
  if (ms == 2) return mk == 2 ? MXK(2, 2) : MXK(2, 3);
  if (ms == 3) return mk == 3 ? MXK(3, 3) : MXK(3, 4);
  return MXK(4, 4);
#undef MXK
}

static const void* mx_fn(const Params& p) {
  const mx::Geo g = mx::make_geo(p);
  const int nch = mx::nch_for(g);
  const int ms = mx::snf_m(g.W), mk = mx::snf_m(g.KW);
  if (p.NP > 2) return nch == 16 ? mx_fn_ms<4, 16>(ms, mk) : nch == 8 ? mx_fn_ms<4, 8>(ms, mk) : mx_fn_ms<4, 4>(ms, mk);
  return nch == 16 ? mx_fn_ms<2, 16>(ms, mk) : nch == 8 ? mx_fn_ms<2, 8>(ms, mk) : mx_fn_ms<2, 4>(ms, mk);
}

cudaError_t launch_mx_kernel(const Params& p, int G, size_t smem, cudaStream_t stream) {
  const void* fn = mx_fn(p);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (G > 8) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.n_traj * G);
  cfg.blockDim = dim3(mx::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  Params pc = p;
  void* args[] = {&pc};
  return cudaLaunchKernelExC(&cfg, fn, args);
}

int mx_max_cluster(const Params& p, size_t smem, int want) {
  const void* fn = mx_fn(p);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (want > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(want);
  cfg.blockDim = dim3(mx::kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = want;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

}  // namespace mpt
