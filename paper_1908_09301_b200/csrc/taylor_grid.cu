// Grid-wide Taylor kernel: ONE trajectory on every SM of the GPU, for the
// large configurations (K = 2200 / 4200 digits, N = 1000 / 3500) whose
// coefficient table (3 (N+1) W digits: up to 21 MB) lives in L2, not in
// shared memory. Persistent cooperative launch (one 256-thread CTA per SM),
// two grid barriers per Taylor order:
//
//   phase A  CTA b: Cauchy terms k = b (mod nblocks) of every pair (rows
//            staged from L2, the newest row from shared memory) and the
//            non-integer linear products; exact column sums reduced in the
//            CTA and added with RED.ADD.64 into the numerator accumulators
//            U_m (already scaled by the integer bilinear coefficients)
//   -- grid barrier --
//   phase B  every CTA: read U_m (L2), add integer linear terms, normalise
//            (redundantly, warp-level) -> U_m digits
//   phase C  CTA b: its share of the (m, column group, p-chunk) items of
//            U_m (x) tau/(i+1) -> RED.ADD.64 into C_m
//   -- grid barrier --
//   phase D  every CTA: normalise C_m -> coefficient i+1 (kept in shared
//            memory; CTA 0 stores it to the L2-resident table)
//
// The arithmetic is the one of oracle/fixmodel.c, bit for bit.
#include <cuda_runtime.h>

#include <cstdint>

#include "mpt_common.cuh"
#include "mpt_device.cuh"

namespace mpt {
namespace grid {

constexpr int kThreads = 512;
constexpr int kPC = 4;

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
  int rw, kc, nrows, nunits, ngmax, ncrow;
  size_t off_stage, off_sinfo, off_crow, off_cinfo, off_part, off_pcar, off_cols, off_ssum, off_xs, off_flag, total;
};

// non-integer linear coefficients get kLinPC partial units each, packed in
// order of appearance (slot = count of non-small entries before it)
constexpr int kLinPC = 4;
__host__ __device__ inline int lin_slot(const Params& p, int it) {
  int s = 0;
  for (int t = 0; t < it; t++) s += p.lin_small[t] ? 0 : 1;
  return s;
}

// phase A k slots: a slot is NP x ceil(NGb/2) lanes, one per (pair q, window
// pair h): each lane accumulates the windows h and NGb-1-h (balanced work)
__host__ __device__ inline int grid_slots(const Params& p, const Geo& g) {
  const int per = (p.NP > 0 ? p.NP : 1) * ((g.NGb + 1) / 2);
  return kThreads / per > 0 ? kThreads / per : 1;
}

// crow: cst D | lin D*D | q NT | ctab | U D | CUR D
__host__ __device__ inline Layout make_layout(const Params& p, int kc) {
  Layout L;
  const Geo g = make_geo(p);
  L.rw = p.RS + 2 * kPad + 1;
  L.kc = kc;
  L.nrows = p.nlv + p.nrv;
  L.ncrow = p.D + p.D * p.D + p.NT + 1 + 2 * p.D;
  const int ns = grid_slots(p, g);
  int nu = ns * (p.NP > 0 ? p.NP : 1) + kLinPC * lin_slot(p, p.D * p.D);
  if (p.D * kPC > nu) nu = p.D * kPC;
  L.nunits = nu;
  L.ngmax = g.NGb;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o += (bytes + 15) / 16 * 16;
    return r;
  };
  L.off_stage = take(sizeof(int32_t) * (size_t)kc * L.nrows * L.rw);
  L.off_sinfo = take(sizeof(int2) * (size_t)kc * L.nrows);
  L.off_crow = take(sizeof(int32_t) * (size_t)L.ncrow * L.rw);
  L.off_cinfo = take(sizeof(int2) * (size_t)L.ncrow);
  L.off_part = take(sizeof(uint32_t) * (size_t)nu * g.NCX);
  L.off_pcar = take(sizeof(int64_t) * (size_t)nu * L.ngmax);
  L.off_cols = take(sizeof(int64_t) * (size_t)(p.NP + 2 * p.D) * g.NCX);
  L.off_ssum = take(sizeof(int64_t) * (size_t)p.D * (p.W + 3));
  L.off_xs = take(sizeof(int64_t) * kMaxD * 32);
  L.off_flag = take(sizeof(int) * 8);
  L.total = o;
  return L;
}

// sense-free generation barrier over the co-resident CTAs of a cooperative launch
__device__ __forceinline__ void grid_barrier(unsigned int* count, unsigned int* gen, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* vgen = gen;
    const unsigned int g0 = *vgen;
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1) {
      *count = 0;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (*vgen == g0) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
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

__device__ __forceinline__ void store_unit(uint32_t* part, int64_t* pcar, const Acc& a, int grp, int c0, int T) {
#pragma unroll
  for (int r = 0; r < kR; r++) {
    const int c = c0 + r - T;
    if (c >= 0) part[c] = (uint32_t)a.v[r];
  }
  pcar[grp] = a.v[kR];
}

__device__ __forceinline__ int64_t unit_col(const uint32_t* part, const int64_t* pcar, int u0, int ustride, int n,
                                            int ncx, int ngmax, int c, int T, int gf, int ng) {
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
    const int64_t* pc = pcar + (size_t)u0 * ngmax + cgb;
#pragma unroll 4
    for (int u = 0; u < n; u++) s += pc[(size_t)u * ustride * ngmax];
  }
  return s;
}

template <int NPT>
__global__ void __launch_bounds__(kThreads, 1) taylor_grid_kernel(const __grid_constant__ Params p, int kc) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Geo g = make_geo(p);
  const Layout L = make_layout(p, kc);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = kThreads / 32;
  const int nb = gridDim.x, b = blockIdx.x;
  const int rw = L.rw;
  int32_t* stage = (int32_t*)(smem + L.off_stage) + kPad;
  int2* stinfo = (int2*)(smem + L.off_sinfo);
  int32_t* crow = (int32_t*)(smem + L.off_crow) + kPad;
  int2* cinfo = (int2*)(smem + L.off_cinfo);
  uint32_t* part = (uint32_t*)(smem + L.off_part);
  int64_t* pcar = (int64_t*)(smem + L.off_pcar);
  int64_t* cols = (int64_t*)(smem + L.off_cols);
  int64_t* ssum = (int64_t*)(smem + L.off_ssum);
  int* flag = (int*)(smem + L.off_flag);
  int64_t* xsb = (int64_t*)(smem + L.off_xs);
  // normalisations: kNW warps per equation (named barrier 1 + m)
  constexpr int kNW = 4;
  const int geq = warp / kNW, gw = warp % kNW;
  auto norm_eq = [&](int m, const int64_t* col, int ncol, int drop, int32_t* out, int2* info, int prec) {
    if (group_normalize(col, ncol, drop, p.W, out, info, prec, gw, kNW, 1 + m, xsb + 32 * m) && gw == 0 && lane == 0)
      flag[0] = 1;
  };
  const int CR_LIN = p.D, CR_Q = CR_LIN + p.D * p.D, CR_CT = CR_Q + p.NT, CR_U = CR_CT + 1, CR_CUR = CR_U + p.D;
  auto CROW = [&](int r) { return crow + (size_t)r * rw; };
  auto SROW = [&](int r) { return stage + (size_t)r * rw; };
  // global scratch: [3 buffers][D][NCX] numerator and coefficient accumulators, barrier words
  unsigned long long* uacc = reinterpret_cast<unsigned long long*>(p.gscratch);
  unsigned long long* cacc = uacc + 3 * (size_t)p.D * g.NCX;
  unsigned int* bar = reinterpret_cast<unsigned int*>(cacc + 3 * (size_t)p.D * g.NCX);
  int32_t* gcoef = p.coef;
  int2* ginfo = p.rinfo;
  auto GROW = [&](int m, int i) { return gcoef + ((size_t)m * (p.N + 1) + i) * p.RS; };
  auto GINF = [&](int m, int i) -> int2& { return ginfo[(size_t)m * (p.N + 1) + i]; };

  for (size_t w = tid; w < L.total / 4; w += kThreads) ((int32_t*)smem)[w] = 0;
  __syncthreads();
  for (int r = 0; r < CR_CT; r++) {
    const int32_t* src = r < CR_LIN ? p.cst + (size_t)r * p.RS
                         : r < CR_Q ? p.lin + (size_t)(r - CR_LIN) * p.RS
                                    : p.q + (size_t)(r - CR_Q) * p.RS;
    for (int d = tid; d < p.W; d += kThreads) CROW(r)[d] = src[d];
  }
  for (int m = 0; m < p.D; m++)
    for (int d = tid; d < p.W; d += kThreads) CROW(CR_CUR + m)[d] = p.state[(size_t)m * p.RS + d];
  __syncthreads();
  for (int r = warp; r < CR_CT; r += nwarps) {
    const int2 inf = row_info_warp(CROW(r), p.W);
    if (lane == 0) cinfo[r] = inf;
  }
  MacCount mcount;
  MacCount* mc = p.counters ? &mcount : nullptr;
  const int nlin = p.D * p.D;
  const int ns = grid_slots(p, g);
  const int NGh = (g.NGb + 1) / 2;
  const int unit_per_slot = (p.NP > 0 ? p.NP : 1) * NGh;
  const int slot = tid / unit_per_slot, urem = tid - slot * unit_per_slot;
  const int qa = urem / NGh, ha = urem - qa * NGh;  // phase A: pair qa, windows ha and NGb-1-ha

  for (int n = p.start_step + 1; n <= p.n_steps; n++) {
    // order 0 rows = state (every CTA holds it; CTA 0 publishes it)
    for (int m = warp; m < p.D; m += nwarps) {
      const int2 inf = row_info_warp(CROW(CR_CUR + m), p.W);
      if (lane == 0) cinfo[CR_CUR + m] = inf;
      for (int d = lane; d < p.W + 3; d += 32) ssum[(size_t)m * (p.W + 3) + d] = d < p.W ? CROW(CR_CUR + m)[d] : 0;
      if (b == 0) {
        for (int d = lane; d < p.RS; d += 32) GROW(m, 0)[d] = d < p.W ? CROW(CR_CUR + m)[d] : 0;
        if (lane == 0) GINF(m, 0) = inf;
      }
    }
    __syncthreads();
    for (int i = 0; i < p.N; i++) {
      const long long gord = (long long)(n - p.start_step - 1) * p.N + i;  // launch-wide order counter
      const bool tlog = p.dbg && n == p.start_step + 1 && b == 0 && tid == 0 && i < 255;
#define TSTAMP(ev) \
  if (tlog) p.dbg[(size_t)(i % 256) * 16 + (ev)] = (long long)clock64();
      TSTAMP(0);
      const int buf = (int)(gord % 3);
      unsigned long long* ua = uacc + (size_t)buf * p.D * g.NCX;
      unsigned long long* ca = cacc + (size_t)buf * p.D * g.NCX;
      // ================= phase A: Cauchy terms k = b (mod nb), staged kc at a time
      if (p.NP > 0) {
        Acc accA, accB;
        acc_zero(accA);
        acc_zero(accB);
        int cntA = 0, cntB = 0;
        const int gB = g.NGb - 1 - ha;
        const bool twoB = gB != ha;
        const int c0A = kR * (g.gfb + ha), c0B = kR * (g.gfb + gB);
        const int nk = b <= i ? (i - b) / nb + 1 : 0;  // this CTA's k values
        // few k values: split every product's p range over several slots
        const int pch = nk > 0 ? max(1, min(16, ns / min(nk, kc))) : 1;
        for (int kk0 = 0; kk0 < nk; kk0 += kc) {
          const int kcn = min(kc, nk - kk0);
          // stage: the newest row (index i) comes from shared memory, older rows from L2
          const int q4 = p.RS / 4;
          for (int e = tid; e < kcn * L.nrows * q4; e += kThreads) {
            const int r = e / q4, w = e - r * q4;
            const int kk = r / L.nrows, v = r - kk * L.nrows;
            const int k = b + (kk0 + kk) * nb;
            const int var = v < p.nlv ? p.lvar[v] : p.rvar[v - p.nlv];
            const int idx = v < p.nlv ? i - k : k;
            int4 v4;
            if (idx == i) {
              const int32_t* s = CROW(CR_CUR + var) + 4 * w;
              v4 = make_int4(s[0], s[1], s[2], s[3]);
            } else {
              v4 = __ldcg(reinterpret_cast<const int4*>(GROW(var, idx)) + w);
            }
            int32_t* dst = SROW(r) + 4 * w;
            dst[0] = v4.x;
            dst[1] = v4.y;
            dst[2] = v4.z;
            dst[3] = v4.w;
          }
          for (int r = tid; r < kcn * L.nrows; r += kThreads) {
            const int kk = r / L.nrows, v = r - kk * L.nrows;
            const int k = b + (kk0 + kk) * nb;
            const int var = v < p.nlv ? p.lvar[v] : p.rvar[v - p.nlv];
            const int idx = v < p.nlv ? i - k : k;
            stinfo[r] = idx == i ? cinfo[CR_CUR + var] : __ldcg(&GINF(var, idx));
          }
          __syncthreads();
          if (slot < ns) {
            for (int wu = slot; wu < kcn * pch; wu += ns) {
              const int kk = wu / pch, pc = wu - kk * pch;
              const int ra = kk * L.nrows + p.pl[qa], rb = kk * L.nrows + p.nlv + p.pr[qa];
              mac_group_chunk(accA, cntA, SROW(ra), stinfo[ra], SROW(rb), stinfo[rb], c0A, g.Tb, pc, pch, mc);
              if (twoB)
                mac_group_chunk(accB, cntB, SROW(ra), stinfo[ra], SROW(rb), stinfo[rb], c0B, g.Tb, pc, pch, mc);
            }
          }
          __syncthreads();
        }
        if (slot < ns) {
          const int u = slot * p.NP + qa;
          acc_fold(accA, c0A, g.Tb);
          store_unit(part + (size_t)u * g.NCX, pcar + (size_t)u * L.ngmax, accA, ha, c0A, g.Tb);
          if (twoB) {
            acc_fold(accB, c0B, g.Tb);
            store_unit(part + (size_t)u * g.NCX, pcar + (size_t)u * L.ngmax, accB, gB, c0B, g.Tb);
          }
        }
      }
      TSTAMP(1);
      // non-integer linear products: item it -> CTA it % nb
      const int nu_a = ns * p.NP;
      // (units nu_a + slot*kLinPC + pc: one product split over kLinPC p-chunks)
      for (int e = tid; e < nlin * g.NGb * kLinPC; e += kThreads) {
        const int it = e / (g.NGb * kLinPC), rem = e - it * g.NGb * kLinPC, grp2 = rem / kLinPC,
                  pc = rem - grp2 * kLinPC;
        if (p.lin_small[it]) continue;
        const int j = it % p.D;
        const int c0 = kR * (g.gfb + grp2);
        Acc acc;
        acc_zero(acc);
        if ((it % nb) == b && cinfo[CR_LIN + it].y >= 0) {
          int cnt = 0;
          mac_group_chunk(acc, cnt, CROW(CR_LIN + it), cinfo[CR_LIN + it], CROW(CR_CUR + j), cinfo[CR_CUR + j], c0,
                          g.Tb, pc, kLinPC, mc);
          acc_fold(acc, c0, g.Tb);
        }
        const int u = nu_a + lin_slot(p, it) * kLinPC + pc;
        store_unit(part + (size_t)u * g.NCX, pcar + (size_t)u * L.ngmax, acc, grp2, c0, g.Tb);
      }
      __syncthreads();
      // CTA column sums -> numerators U_m (integer q applied) -> RED.ADD.64
      const int nkall = b <= i ? (i - b) / nb + 1 : 0;
      const int nsa = nkall > 0 ? ns : 0;  // every slot may hold a p-chunk
      for (int w = tid; w < p.D * g.ncolb; w += kThreads) {
        const int m = w / g.ncolb, c = w - m * g.ncolb;
        int64_t s = 0;
        if (nsa > 0)
          for (int t = 0; t < p.NT; t++)
            if (p.teq[t] == m)
              s += (int64_t)p.tq_int[t] *
                   unit_col(part, pcar, p.tpair[t], p.NP, nsa, g.NCX, L.ngmax, c, g.Tb, g.gfb, g.NGb);
        for (int j = 0; j < p.D; j++)
          if (!p.lin_small[m * p.D + j] && ((m * p.D + j) % nb) == b)
            s += unit_col(part, pcar, nu_a + lin_slot(p, m * p.D + j) * kLinPC, 1, kLinPC, g.NCX, L.ngmax, c, g.Tb, g.gfb, g.NGb);
        if (s != 0) atomicAdd(&ua[(size_t)m * g.NCX + c], (unsigned long long)s);
      }
      TSTAMP(2);
      grid_barrier(bar, bar + 1, nb);
      TSTAMP(3);
      // ================= phase B: numerators (redundant in every CTA)
      if (b == 0) {  // recycle the buffers of the next order (last read three orders ago)
        unsigned long long* nu2 = uacc + (size_t)((gord + 1) % 3) * p.D * g.NCX;
        unsigned long long* nc2 = cacc + (size_t)((gord + 1) % 3) * p.D * g.NCX;
        for (int w = tid; w < p.D * g.NCX; w += kThreads) {
          nu2[w] = 0;
          nc2[w] = 0;
        }
      }
      int64_t* ucol = cols + (size_t)p.NP * g.NCX;
      int64_t* ccol = ucol + (size_t)p.D * g.NCX;
      for (int d = tid; d < p.W; d += kThreads) CROW(CR_CT)[d] = __ldg(p.ctab + (size_t)i * p.RS + d);
      for (int w = tid; w < p.D * g.ncolb; w += kThreads) {
        const int m = w / g.ncolb, c = w - m * g.ncolb;
        int64_t s = (int64_t)__ldcg(&ua[(size_t)m * g.NCX + c]);
        if (c >= 2 && c - 2 < p.W) {
          const int dgt = c - 2;
          if (i == 0) s += CROW(m)[dgt];
          for (int j = 0; j < p.D; j++)
            if (p.lin_small[m * p.D + j]) s += (int64_t)p.lin_int[m * p.D + j] * CROW(CR_CUR + j)[dgt];
        }
        ucol[(size_t)m * g.NCX + c] = s;
      }
      __syncthreads();
      TSTAMP(4);
      if (geq < p.D) norm_eq(geq, ucol + (size_t)geq * g.NCX, g.ncolb, 2, CROW(CR_U + geq), &cinfo[CR_U + geq], 0);
      if (warp == nwarps - 1) {
        const int2 inf = row_info_warp(CROW(CR_CT), p.W);
        if (lane == 0) cinfo[CR_CT] = inf;
      }
      __syncthreads();
      TSTAMP(5);
      // ================= phase C: this CTA's share of U_m (x) tau/(i+1)
      {
        const int nitems = p.D * g.NGc * kPC;
        for (int e = tid; e < p.D * kPC * g.NGc; e += kThreads) {
          // every local thread slot writes its unit (zeros when it has no item)
          const int m = e / (g.NGc * kPC), rem = e - m * g.NGc * kPC, gg = rem / kPC, pc = rem - gg * kPC;
          const int item = e;  // global item id
          const int c0 = kR * (g.gfc + gg);
          Acc acc;
          acc_zero(acc);
          if ((item % nb) == b) {
            int2 ia = cinfo[CR_U + m];
            const int2 ib = cinfo[CR_CT];
            const int plo = max(ia.x, c0 - ib.y), phi = min(ia.y, c0 + kR - 1 - ib.x);
            if (plo <= phi) {
              const int b0 = plo / kR, nbk = phi / kR - b0 + 1;
              const int per = (nbk + kPC - 1) / kPC;
              const int blo = b0 + pc * per, bhi = min(b0 + nbk, blo + per) - 1;
              if (blo <= bhi) {
                ia.x = max(ia.x, blo * kR);
                ia.y = min(ia.y, bhi * kR + kR - 1);
                int cnt = 0;
                mac_group(acc, cnt, CROW(CR_U + m), ia, CROW(CR_CT), ib, c0, g.Tc, mc);
                acc_fold(acc, c0, g.Tc);
              }
            }
          }
          const int u = m * kPC + pc;
          store_unit(part + (size_t)u * g.NCX, pcar + (size_t)u * L.ngmax, acc, gg, c0, g.Tc);
        }
        (void)nitems;
        __syncthreads();
        for (int w = tid; w < p.D * g.ncolc; w += kThreads) {
          const int m = w / g.ncolc, c = w - m * g.ncolc;
          const int64_t s = unit_col(part, pcar, m * kPC, 1, kPC, g.NCX, L.ngmax, c, g.Tc, g.gfc, g.NGc);
          if (s != 0) atomicAdd(&ca[(size_t)m * g.NCX + c], (unsigned long long)s);
        }
      }
      TSTAMP(6);
      grid_barrier(bar, bar + 1, nb);
      TSTAMP(7);
      // ================= phase D: coefficient i+1 (redundant), CTA 0 publishes
      for (int w = tid; w < p.D * g.ncolc; w += kThreads) {
        const int m = w / g.ncolc, c = w - m * g.ncolc;
        ccol[(size_t)m * g.NCX + c] = (int64_t)__ldcg(&ca[(size_t)m * g.NCX + c]);
      }
      __syncthreads();
      if (geq < p.D) norm_eq(geq, ccol + (size_t)geq * g.NCX, g.ncolc, 2, CROW(CR_CUR + geq), &cinfo[CR_CUR + geq], 0);
      __syncthreads();
      TSTAMP(8);
      for (int m = warp; m < p.D; m += nwarps) {
        for (int d = lane; d < p.W; d += 32) ssum[(size_t)m * (p.W + 3) + d] += CROW(CR_CUR + m)[d];
        if (b == 0) {
          for (int d = lane; d < p.RS; d += 32) GROW(m, i + 1)[d] = d < p.W ? CROW(CR_CUR + m)[d] : 0;
          if (lane == 0) GINF(m, i + 1) = cinfo[CR_CUR + m];
        }
      }
      __syncthreads();
      TSTAMP(9);
#undef TSTAMP
    }
    // state = RN_P(sum of the rows)
    if (geq < p.D) norm_eq(geq, ssum + (size_t)geq * (p.W + 3), p.W + 3, 0, CROW(CR_CUR + geq), &cinfo[CR_CUR + geq], p.P);
    __syncthreads();
    if (b == 0 && ((n % p.stride == 0) || (n == p.n_steps))) {
      const int slot2 = (n % p.stride == 0) ? (n / p.stride - p.start_step / p.stride)
                                            : (p.n_steps / p.stride - p.start_step / p.stride + 1);
      int32_t* dst = p.rec + (size_t)slot2 * p.D * p.RS;
      for (int m = 0; m < p.D; m++)
        for (int d = tid; d < p.W; d += kThreads) dst[(size_t)m * p.RS + d] = CROW(CR_CUR + m)[d];
    }
    // the next step's order 0 reads row 0 from L2 only at orders >= 1 (after barriers)
  }
  if (b == 0) {
    for (int m = 0; m < p.D; m++)
      for (int d = tid; d < p.W; d += kThreads) p.state[(size_t)m * p.RS + d] = CROW(CR_CUR + m)[d];
  }
  __syncthreads();
  if (tid == 0 && flag[0]) atomicOr(p.status, kOverflow);
  if (mc) {
    atomicAdd(&p.counters[0], mcount.useful);
    atomicAdd(&p.counters[1], mcount.executed);
  }
}

}  // namespace grid

bool grid_supported(const Params& p) { return p.n_traj == 1 && p.all_q_small; }

size_t grid_smem_bytes(const Params& p, int kc) { return grid::make_layout(p, kc).total; }

size_t grid_scratch_bytes(const Params& p) {
  const grid::Geo g = grid::make_geo(p);
  return sizeof(unsigned long long) * 6 * (size_t)p.D * g.NCX + 64;
}

cudaError_t launch_grid_kernel(const Params& p, int nblocks, int kc, size_t smem, cudaStream_t stream) {
  const int npt = p.NP <= 1 ? 1 : p.NP <= 2 ? 2 : 4;
  const void* fn = npt == 1 ? (const void*)grid::taylor_grid_kernel<1>
                   : npt == 2 ? (const void*)grid::taylor_grid_kernel<2>
                              : (const void*)grid::taylor_grid_kernel<4>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  Params pc = p;
  int kcc = kc;
  void* args[] = {&pc, &kcc};
  return cudaLaunchCooperativeKernel(fn, dim3(nblocks), dim3(grid::kThreads), args, smem, stream);
}

int grid_max_blocks(const Params& p, size_t smem) {
  const void* fn = (const void*)grid::taylor_grid_kernel<2>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, grid::kThreads, smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return per_sm * sms;
}

}  // namespace mpt
