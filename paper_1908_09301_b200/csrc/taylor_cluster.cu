// Shared-memory-resident persistent Taylor kernel: one thread-block CLUSTER
// of G CTAs (G = 1..16) integrates one trajectory for the whole launch.
//
// Every CTA keeps the coefficient rows it needs in shared memory for the
// whole step (no per-order restaging) and recomputes the small per-order
// "chain" (numerators, tau/(i+1) scaling, normalisation) redundantly, so all
// CTAs hold bit-identical new coefficients without a second exchange. The
// only per-order communication is the Cauchy-sum partials:
//
//   phase A  CTA r accumulates sum_k coef[j_p][i-k] (x) coef[k_p][k] for its
//            k = r (mod G) (plus non-integer linear terms) into exact int64
//            column registers, then smem atomics into its exchange buffer;
//   ---- one cluster barrier (barrier.cluster arrive.release / wait.acquire)
//   phase B  every CTA sums the G exchange buffers over DSMEM
//            (ld.shared::cluster), forms the numerators U_m, normalises them;
//   phase C  coef[m][i+1] = rnd(U_m (x) tau/(i+1)), split over the CTA.
//
// Rows of "left" factors (the a_{i-k} side: needed at every index) are kept
// in full; rows used only as right factors are kept for the CTA's own k
// residue class. State sums (the fused, tau-scaled Horner evaluation) are
// accumulated as each coefficient is created. Arithmetic = oracle/fixmodel.c.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "mpt_common.cuh"
#include "mpt_device.cuh"

namespace cg = cooperative_groups;

namespace mpt {
namespace cl {

constexpr int kThreads = 256;
constexpr int kPC = 4;  // p-range split of the tau/(i+1) products

struct Geo {
  int Tb, gfb, NGb, Tc, gfc, NGc, NCX, ncolb, ncolc;
};

__host__ __device__ inline Geo make_geo(const Params& p) {
  Geo g;
  g.Tb = p.Lf - 2;
  g.gfb = g.Tb / kR;
  g.NGb = (2 * p.Lf) / kR - g.gfb + 1;
  g.Tc = p.Lf + p.sc - 2;
  g.gfc = g.Tc / kR;
  g.NGc = (2 * p.Lf) / kR - g.gfc + 1;
  g.NCX = kR * (g.NGb + 2);
  g.ncolb = kR * (g.gfb + g.NGb) - g.Tb + 1;
  g.ncolc = kR * (g.gfc + g.NGc) - g.Tc + 1;
  return g;
}

struct Layout {
  int rs;        // words per row slot (W rounded to 4, plus kPad zero gap)
  int nslots;    // coefficient row slots
  int base[kMaxD], full[kMaxD];  // per variable: first slot, 1 = every index kept
  int ncrow;     // constant rows: cst D, lin D*D, q NT, ctab 1, U D, S NP, cur D
  int ntg;       // exchange targets: NP pair sums + D linear-product sums
  int nunits;    // partial-sum units (one writer per (unit, column group))
  int ngmax;     // column groups per unit
  size_t off_rows, off_rinfo, off_crow, off_cinfo, off_xbuf, off_cols, off_ssum, off_part, off_pcar, off_utg,
      off_flag, total;
};

// rows: a variable that appears as a left factor keeps all N+1 indices; a
// variable used only as a right factor (or not at all) keeps the indices
// k = rank (mod G).
__host__ __device__ inline Layout make_layout(const Params& p, int G) {
  Layout L;
  L.rs = (p.W + 3) / 4 * 4 + kPad + 1;  // odd: k-slots hit different banks
  int s = 0;
  for (int v = 0; v < p.D; v++) {
    int is_left = 0;
    for (int q = 0; q < p.NP; q++) is_left |= (p.pj[q] == v);
    L.full[v] = is_left || G == 1;
    L.base[v] = s;
    s += L.full[v] ? p.N + 1 : (p.N + G) / G;
  }
  L.nslots = s;
  L.ncrow = p.D + p.D * p.D + p.NT + 1 + p.D + (p.NP > 0 ? p.NP : 1) + p.D;
  L.ntg = p.NP + p.D;
  Geo g = make_geo(p);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o += (bytes + 15) / 16 * 16;
    return r;
  };
  L.off_rows = take(sizeof(int32_t) * ((size_t)L.nslots * L.rs + kPad));
  L.off_rinfo = take(sizeof(int2) * (size_t)L.nslots);
  L.off_crow = take(sizeof(int32_t) * ((size_t)L.ncrow * L.rs + kPad));
  L.off_cinfo = take(sizeof(int2) * (size_t)L.ncrow);
  L.off_xbuf = take(sizeof(int64_t) * 2 * (size_t)L.ntg * g.NCX);
  L.off_cols = take(sizeof(int64_t) * (size_t)(L.ntg + p.D) * g.NCX);
  L.off_ssum = take(sizeof(int64_t) * (size_t)p.D * (p.W + 3));
  const int ns = kThreads / g.NGb;
  int nu = ns * (p.NP > 0 ? p.NP : 1) + p.D * p.D;
  if (p.NT > nu) nu = p.NT;
  if (p.D * kPC > nu) nu = p.D * kPC;
  L.nunits = nu;
  L.ngmax = g.NGb > g.NGc ? g.NGb : g.NGc;
  L.off_part = take(sizeof(uint32_t) * (size_t)nu * g.NCX);
  L.off_pcar = take(sizeof(int64_t) * (size_t)nu * L.ngmax);
  L.off_utg = take(sizeof(int) * (size_t)nu);
  L.off_flag = take(sizeof(int) * 8);
  L.total = o;
  return L;
}

__device__ __forceinline__ int2 row_info_warp(const int32_t* row, int W) {
  int bot = 1 << 30, tp = -1;
  for (int d = threadIdx.x & 31; d < W; d += 32)
    if (row[d]) {
      bot = min(bot, d);
      tp = max(tp, d);
    }
  bot = __reduce_min_sync(0xffffffffu, bot);
  tp = __reduce_max_sync(0xffffffffu, tp);
  return make_int2(tp >= 0 ? bot : W, tp);
}

// one writer per (unit, group): the folded digits (in [0, B)) of the group's
// columns and the group's carry into the next group's first column
__device__ __forceinline__ void store_unit(uint32_t* part, int64_t* pcar, const Acc& a, int grp, int c0, int T) {
#pragma unroll
  for (int r = 0; r < kR; r++) {
    const int c = c0 + r - T;
    if (c >= 0) part[c] = (uint32_t)a.v[r];
  }
  pcar[grp] = a.v[kR];
}

// column c (relative to T) of a target whose units are u0, u0 + ustride, ...
// (n units): folded digits of the group that owns the column plus the carry
// of the group below it
__device__ __forceinline__ int64_t strided_sum(const uint32_t* part, const int64_t* pcar, int u0, int ustride, int n,
                                               int ncx, int ngmax, int c, int T, int gf, int ng) {
  const int cabs = c + T;
  const int own = cabs / kR - gf;
  const int cg = (cabs % kR == 0) ? cabs / kR - 1 - gf : -1;
  int64_t s = 0;
  if (own >= 0 && own < ng) {
    const uint32_t* pp = part + (size_t)u0 * ncx + c;
    const size_t st = (size_t)ustride * ncx;
#pragma unroll 4
    for (int u = 0; u < n; u++) s += pp[u * st];
  }
  if (cg >= 0 && cg < ng) {
    const int64_t* pc = pcar + (size_t)u0 * ngmax + cg;
    const size_t st = (size_t)ustride * ngmax;
#pragma unroll 4
    for (int u = 0; u < n; u++) s += pc[u * st];
  }
  return s;
}

template <int NPT>
__global__ void __launch_bounds__(kThreads, 1) taylor_cluster_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(16) unsigned char smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int G = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int traj = blockIdx.x / G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = kThreads / 32;
  const Geo g = make_geo(p);
  const Layout L = make_layout(p, G);

  int32_t* rows = (int32_t*)(smem + L.off_rows) + kPad;
  int2* rinfo = (int2*)(smem + L.off_rinfo);
  int32_t* crow = (int32_t*)(smem + L.off_crow) + kPad;
  int2* cinfo = (int2*)(smem + L.off_cinfo);
  int64_t* xbuf = (int64_t*)(smem + L.off_xbuf);
  int64_t* cols = (int64_t*)(smem + L.off_cols);
  int64_t* ssum = (int64_t*)(smem + L.off_ssum);
  uint32_t* part = (uint32_t*)(smem + L.off_part);
  int64_t* pcar = (int64_t*)(smem + L.off_pcar);
  int* flag = (int*)(smem + L.off_flag);
  const int rs = L.rs;
  // constant-row indices
  const int CR_CST = 0, CR_LIN = p.D, CR_Q = p.D + p.D * p.D, CR_CT = CR_Q + p.NT, CR_U = CR_CT + 1,
            CR_S = CR_U + p.D, CR_CUR = CR_S + (p.NP > 0 ? p.NP : 1);
  auto CROW = [&](int r) { return crow + (size_t)r * rs; };
  __shared__ int s_base[kMaxD], s_full[kMaxD];
  if (tid < kMaxD) {
    s_base[tid] = tid < p.D ? L.base[tid] : 0;
    s_full[tid] = tid < p.D ? L.full[tid] : 1;
  }
  __shared__ const int64_t* s_remote[16];  // DSMEM views of every cluster CTA's exchange buffers
  if (tid < 16) s_remote[tid] = tid < G ? cluster.map_shared_rank(xbuf, tid) : nullptr;
  auto has_row = [&](int v, int k) { return s_full[v] || (k % G) == rank; };
  auto SLOT = [&](int v, int k) { return s_base[v] + (s_full[v] ? k : k / G); };
  auto ROW = [&](int v, int k) { return rows + (size_t)SLOT(v, k) * rs; };

  for (size_t w = tid; w < L.total / 4; w += kThreads) ((int32_t*)smem)[w] = 0;
  __syncthreads();

  // constants
  for (int r = 0; r < CR_CT; r++) {
    const int32_t* src = r < CR_LIN ? p.cst + (size_t)r * p.RS
                         : r < CR_Q ? p.lin + (size_t)(r - CR_LIN) * p.RS
                                    : p.q + (size_t)(r - CR_Q) * p.RS;
    for (int d = tid; d < p.W; d += kThreads) CROW(r)[d] = src[d];
  }
  int32_t* gstate = p.state + (size_t)traj * p.D * p.RS;
  for (int m = 0; m < p.D; m++)
    for (int d = tid; d < p.W; d += kThreads) CROW(CR_CUR + m)[d] = gstate[(size_t)m * p.RS + d];
  __syncthreads();
  for (int r = warp; r < CR_CT; r += nwarps) {
    int2 inf = row_info_warp(CROW(r), p.W);
    if (lane == 0) cinfo[r] = inf;
  }

  MacCount mcount;
  MacCount* mc = p.counters ? &mcount : nullptr;
  // phase-A mapping: which linear products are real products (not small ints)
  const int nlin = p.D * p.D;

  for (int n = p.start_step + 1; n <= p.n_steps; n++) {
    // ---- order-0 rows = state; state column sums start with them
    for (int m = 0; m < p.D; m++) {
      const int32_t* cur = CROW(CR_CUR + m);
      for (int d = tid; d < p.W + 3; d += kThreads) ssum[(size_t)m * (p.W + 3) + d] = d < p.W ? cur[d] : 0;
      if (has_row(m, 0))
        for (int d = tid; d < p.W; d += kThreads) ROW(m, 0)[d] = cur[d];
    }
    __syncthreads();
    for (int m = warp; m < p.D; m += nwarps) {
      int2 inf = row_info_warp(CROW(CR_CUR + m), p.W);
      if (lane == 0) {
        cinfo[CR_CUR + m] = inf;
        if (has_row(m, 0)) rinfo[SLOT(m, 0)] = inf;
      }
    }
    if (p.write_coef && rank == 0)
      for (int m = 0; m < p.D; m++)
        for (int d = tid; d < p.W; d += kThreads)
          p.coef[(((size_t)traj * p.D + m) * (p.N + 1)) * p.RS + d] = CROW(CR_CUR + m)[d];
    __syncthreads();

    for (int i = 0; i < p.N; i++) {
      int64_t* xb = xbuf + (size_t)(i & 1) * L.ntg * g.NCX;
      // tau/(i+1) row: issue the loads early, used in phase C
      for (int d = tid; d < p.W; d += kThreads) CROW(CR_CT)[d] = __ldg(p.ctab + (size_t)i * p.RS + d);
      // ================= phase A: Cauchy partial sums for k = rank (mod G)
      {
        const int ns = kThreads / g.NGb;
        const int slot = tid / g.NGb, grp = tid - slot * g.NGb;
        const int nu_a = ns * p.NP;
        const int nk = rank <= i ? (i - rank) / G + 1 : 0;
        const int nsa = min(ns, nk);  // slots with work this order
        if (slot < nsa) {
          const int c0 = kR * (g.gfb + grp);
          Acc acc[NPT];
          int cnt[NPT];
#pragma unroll
          for (int q = 0; q < NPT; q++) {
            acc_zero(acc[q]);
            cnt[q] = 0;
          }
          for (int kk = slot; kk < nk; kk += ns) {
            const int k = rank + kk * G;
#pragma unroll
            for (int q = 0; q < NPT; q++) {
              if (q < p.NP) {
                const int va = p.pj[q], vb = p.pk[q];
                mac_group(acc[q], cnt[q], ROW(va, i - k), rinfo[SLOT(va, i - k)], ROW(vb, k), rinfo[SLOT(vb, k)], c0,
                          g.Tb, mc);
              }
            }
          }
#pragma unroll
          for (int q = 0; q < NPT; q++) {
            if (q < p.NP) {
              acc_fold(acc[q], c0, g.Tb);
              const int u = slot * p.NP + q;
              store_unit(part + (size_t)u * g.NCX, pcar + (size_t)u * L.ngmax, acc[q], grp, c0, g.Tb);
            }
          }
        }
        // linear terms with non-small-integer coefficients: item it -> CTA it % G
        for (int e = tid; e < nlin * g.NGb; e += kThreads) {
          const int it = e / g.NGb, grp2 = e - it * g.NGb;
          if (p.lin_small[it]) continue;
          const int m = it / p.D, j = it - m * p.D;
          const int c0 = kR * (g.gfb + grp2);
          Acc acc;
          acc_zero(acc);
          if ((it % G) == rank && cinfo[CR_LIN + it].y >= 0) {
            int cnt = 0;
            mac_group(acc, cnt, CROW(CR_LIN + it), cinfo[CR_LIN + it], CROW(CR_CUR + j), cinfo[CR_CUR + j], c0, g.Tb,
                      mc);
            acc_fold(acc, c0, g.Tb);
          }
          const int u = nu_a + it;
          store_unit(part + (size_t)u * g.NCX, pcar + (size_t)u * L.ngmax, acc, grp2, c0, g.Tb);
        }
        __syncthreads();
        // this CTA's exchange buffer: per target column sums over its units
        for (int w = tid; w < L.ntg * g.ncolb; w += kThreads) {
          const int tg = w / g.ncolb, c = w - tg * g.ncolb;
          int64_t s = 0;
          if (tg < p.NP) {
            s = strided_sum(part, pcar, tg, p.NP, nsa, g.NCX, L.ngmax, c, g.Tb, g.gfb, g.NGb);
          } else if (p.tg_used[tg]) {
            const int m = tg - p.NP;
            for (int j = 0; j < p.D; j++)
              if (!p.lin_small[m * p.D + j])
                s += strided_sum(part, pcar, nu_a + m * p.D + j, 1, 1, g.NCX, L.ngmax, c, g.Tb, g.gfb, g.NGb);
          }
          xb[(size_t)tg * g.NCX + c] = s;
        }
      }
      __syncthreads();
      // ================= exchange: one cluster barrier, then DSMEM gather
      cluster.sync();
      for (int w = tid; w < L.ntg * g.ncolb; w += kThreads) {
        const int tg = w / g.ncolb, c = w - tg * g.ncolb;
        const size_t off = (size_t)(i & 1) * L.ntg * g.NCX + (size_t)tg * g.NCX + c;
        int64_t s = 0;
        if (!p.tg_used[tg]) {
          cols[(size_t)tg * g.NCX + c] = 0;
          continue;
        }
        // all G remote loads in flight before the first use
        int64_t v[16];
#pragma unroll
        for (int rr = 0; rr < 16; rr++) v[rr] = rr < G ? s_remote[rr][off] : 0;
#pragma unroll
        for (int rr = 0; rr < 16; rr++) s += v[rr];
        cols[(size_t)tg * g.NCX + c] = s;
      }
      __syncthreads();
      // ================= phase B: numerators
      // (general path) pairs used by non-integer q terms are rounded first
      for (int q = warp; q < p.NP; q += nwarps) {
        if (!p.pair_round[q]) continue;
        if (warp_normalize(cols + (size_t)q * g.NCX, g.ncolb, 2, p.W, CROW(CR_S + q), &cinfo[CR_S + q], 0) &&
            lane == 0)
          flag[0] = 1;
      }
      __syncthreads();
      int64_t* ucol = cols + (size_t)L.ntg * g.NCX;
      for (int w = tid; w < p.D * g.ncolb; w += kThreads) {
        const int m = w / g.ncolb, c = w - m * g.ncolb;
        int64_t s = cols[(size_t)(p.NP + m) * g.NCX + c];
        if (c >= 2 && c - 2 < p.W) {
          const int dgt = c - 2;
          if (i == 0) s += CROW(CR_CST + m)[dgt];
          for (int j = 0; j < p.D; j++)
            if (p.lin_small[m * p.D + j]) s += (int64_t)p.lin_int[m * p.D + j] * CROW(CR_CUR + j)[dgt];
        }
        for (int t = 0; t < p.NT; t++)
          if (p.teq[t] == m && p.tq_small[t]) s += (int64_t)p.tq_int[t] * cols[(size_t)p.tpair[t] * g.NCX + c];
        ucol[(size_t)m * g.NCX + c] = s;
      }
      __syncthreads();
      // non-integer q terms: tprod(q_t, S_p) (general systems only)
      if (p.NP > 0 && !p.all_q_small) {
        for (int e = tid; e < p.NT * g.NGb; e += kThreads) {
          const int t = e / g.NGb, grp = e - t * g.NGb;
          const int c0 = kR * (g.gfb + grp);
          Acc acc;
          acc_zero(acc);
          if (!p.tq_small[t]) {
            int cnt = 0;
            mac_group(acc, cnt, CROW(CR_Q + t), cinfo[CR_Q + t], CROW(CR_S + p.tpair[t]), cinfo[CR_S + p.tpair[t]],
                      c0, g.Tb, mc);
            acc_fold(acc, c0, g.Tb);
          }
          store_unit(part + (size_t)t * g.NCX, pcar + (size_t)t * L.ngmax, acc, grp, c0, g.Tb);
        }
        __syncthreads();
        for (int w = tid; w < p.D * g.ncolb; w += kThreads) {
          const int m = w / g.ncolb, c = w - m * g.ncolb;
          for (int t = 0; t < p.NT; t++)
            if (p.teq[t] == m && !p.tq_small[t])
              ucol[(size_t)m * g.NCX + c] += strided_sum(part, pcar, t, 1, 1, g.NCX, L.ngmax, c, g.Tb, g.gfb, g.NGb);
        }
        __syncthreads();
      }
      for (int m = warp; m < p.D; m += nwarps) {
        if (warp_normalize(ucol + (size_t)m * g.NCX, g.ncolb, 2, p.W, CROW(CR_U + m), &cinfo[CR_U + m], 0) && lane == 0)
          flag[0] = 1;
      }
      if (warp == nwarps - 1) {
        int2 inf = row_info_warp(CROW(CR_CT), p.W);
        if (lane == 0) cinfo[CR_CT] = inf;
      }
      __syncthreads();
      // ================= phase C: coef[m][i+1] = rnd(U_m (x) tau/(i+1))
      for (int e = tid; e < p.D * g.NGc * kPC; e += kThreads) {
        const int m = e / (g.NGc * kPC), rem = e - m * g.NGc * kPC, grp = rem / kPC, pc = rem - grp * kPC;
        const int c0 = kR * (g.gfc + grp);
        int2 ia = cinfo[CR_U + m];
        const int2 ib = cinfo[CR_CT];
        Acc acc;
        acc_zero(acc);
        // split the p range of this group into kPC chunks of whole kR blocks
        const int plo = max(ia.x, c0 - ib.y), phi = min(ia.y, c0 + kR - 1 - ib.x);
        if (plo <= phi) {
          const int b0 = plo / kR, nb = phi / kR - b0 + 1;
          const int per = (nb + kPC - 1) / kPC;
          const int blo = b0 + pc * per, bhi = min(b0 + nb, blo + per) - 1;
          if (blo <= bhi) {
            ia.x = max(ia.x, blo * kR);
            ia.y = min(ia.y, bhi * kR + kR - 1);
            int cnt = 0;
            mac_group(acc, cnt, CROW(CR_U + m), ia, CROW(CR_CT), ib, c0, g.Tc, mc);
            acc_fold(acc, c0, g.Tc);
          }
        }
        const int u = m * kPC + pc;
        store_unit(part + (size_t)u * g.NCX, pcar + (size_t)u * L.ngmax, acc, grp, c0, g.Tc);
      }
      __syncthreads();
      for (int w = tid; w < p.D * g.ncolc; w += kThreads) {
        const int m = w / g.ncolc, c = w - m * g.ncolc;
        ucol[(size_t)m * g.NCX + c] = strided_sum(part, pcar, m * kPC, 1, kPC, g.NCX, L.ngmax, c, g.Tc, g.gfc, g.NGc);
      }
      __syncthreads();
      for (int m = warp; m < p.D; m += nwarps) {
        if (warp_normalize(ucol + (size_t)m * g.NCX, g.ncolc, 2, p.W, CROW(CR_CUR + m), &cinfo[CR_CUR + m], 0) &&
            lane == 0)
          flag[0] = 1;
      }
      __syncthreads();
      // store the new coefficients where they are needed and add them to the state sums
      for (int m = 0; m < p.D; m++) {
        const int32_t* cur = CROW(CR_CUR + m);
        const bool keep = has_row(m, i + 1);
        for (int d = tid; d < p.W; d += kThreads) {
          ssum[(size_t)m * (p.W + 3) + d] += cur[d];
          if (keep) ROW(m, i + 1)[d] = cur[d];
        }
        if (keep && tid == 0) rinfo[SLOT(m, i + 1)] = cinfo[CR_CUR + m];
        if (p.write_coef && rank == 0) {
          int32_t* dst = p.coef + (((size_t)traj * p.D + m) * (p.N + 1) + i + 1) * p.RS;
          for (int d = tid; d < p.W; d += kThreads) dst[d] = cur[d];
        }
      }
      __syncthreads();
    }
    // ---- state = RN_P(sum_i coef[m][i]) (exact sum; drop = 0), identical in every CTA
    for (int m = warp; m < p.D; m += nwarps) {
      if (warp_normalize(ssum + (size_t)m * (p.W + 3), p.W + 3, 0, p.W, CROW(CR_CUR + m), &cinfo[CR_CUR + m], p.P) &&
          lane == 0)
        flag[0] = 1;
    }
    __syncthreads();
    if (rank == 0 && ((n % p.stride == 0) || (n == p.n_steps))) {
      const int slot = (n % p.stride == 0) ? (n / p.stride - p.start_step / p.stride)
                                           : (p.n_steps / p.stride - p.start_step / p.stride + 1);
      int32_t* dst = p.rec + ((size_t)slot * p.n_traj + traj) * p.D * p.RS;
      for (int m = 0; m < p.D; m++)
        for (int d = tid; d < p.W; d += kThreads) dst[(size_t)m * p.RS + d] = CROW(CR_CUR + m)[d];
    }
  }
  if (rank == 0) {
    for (int m = 0; m < p.D; m++)
      for (int d = tid; d < p.W; d += kThreads) gstate[(size_t)m * p.RS + d] = CROW(CR_CUR + m)[d];
  }
  __syncthreads();
  if (rank == 0 && tid == 0) p.status[traj] = flag[0] ? kOverflow : kOk;
  if (mc) {
    atomicAdd(&p.counters[0], mcount.useful);
    atomicAdd(&p.counters[1], mcount.executed);
  }
  cluster.sync();  // no CTA may exit while others can still read its shared memory
}

}  // namespace cl

size_t cluster_smem_bytes(const Params& p, int G) { return cl::make_layout(p, G).total; }

cudaError_t launch_cluster_kernel(const Params& p, int G, size_t smem, cudaStream_t stream) {
  const int npt = p.NP <= 1 ? 1 : p.NP <= 2 ? 2 : p.NP <= 4 ? 4 : 8;
  const void* fn = npt == 1   ? (const void*)cl::taylor_cluster_kernel<1>
                   : npt == 2 ? (const void*)cl::taylor_cluster_kernel<2>
                   : npt == 4 ? (const void*)cl::taylor_cluster_kernel<4>
                              : (const void*)cl::taylor_cluster_kernel<8>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (G > 8) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.n_traj * G);
  cfg.blockDim = dim3(cl::kThreads);
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

// largest cluster the device can co-schedule for this kernel and smem size
int max_cluster_size(const Params& p, size_t smem, int want) {
  const void* fn = (const void*)cl::taylor_cluster_kernel<2>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (want > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(want);
  cfg.blockDim = dim3(cl::kThreads);
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
