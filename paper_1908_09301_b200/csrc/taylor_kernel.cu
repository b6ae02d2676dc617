// Persistent multiple-precision Taylor kernel for sm_100a.
//
// One CTA owns one trajectory for the whole launch: it loops over steps and,
// inside each step, over the Taylor orders i = 0..N-1 of the recurrence
// (reference taylor.py:117 _jet_rows, paper Eq. (3)), with __syncthreads()
// between phases instead of kernel relaunches. Per order:
//
//   phase A  Cauchy sums  S_p = sum_k coef[j_p][i-k] (x) coef[k_p][k]
//            column-wise in exact 64-bit integer accumulators (IMAD.WIDE),
//            rows staged in shared memory, leading/trailing zero digits
//            skipped, ONE carry propagation + rounding per sum.
//   phase B  numerators U_m = [i==0] c_m + sum_j L_mj (x) coef[j][i]
//                             + sum_t q_t (x) S_{p_t}
//   phase C  coef[m][i+1] = U_m (x) tau/(i+1)       (the 1/(i+1) scaling)
//
// and after the last order the state update x_{n+1} = sum_i coef[i] (the
// tau-scaled Horner evaluation, reference taylor.py:168) followed by the
// rounding of the state to the reference precision P (round-to-nearest-even).
// oracle/fixmodel.c restates exactly this arithmetic on the CPU.
#include <cuda_runtime.h>

#include <cstdint>

#include "mpt_common.cuh"
#include "mpt_device.cuh"

namespace mpt {

__host__ __device__ inline int round_up(int x, int m) { return (x + m - 1) / m * m; }
// odd row stride: consecutive k-slots fall into different shared-memory banks
__host__ __device__ inline int row_words(int RS) { return RS + 2 * kPad + 1; }

struct Geo {
  int Tb, gfb, NGb;  // base products: first column, first group, #groups
  int Tc, gfc, NGc;  // tau/(i+1) products
  int NCX;           // column-sum length (relative to T), covers all groups + carry
};

// Phase A partial columns: one padding slot after every 8 columns and an odd unit
// stride, so the lanes of a warp (8-column windows 64 bytes apart, units NCX
// apart) spread over the shared-memory banks instead of piling on two of them.
__host__ __device__ inline int part_idx(int c) { return c + (c >> 3); }
__host__ __device__ inline int part_stride(int NCX) { return (NCX + NCX / 8 + 1) | 1; }

__host__ __device__ inline Geo make_geo(const Params& p) {
  Geo g;
  g.Tb = p.Lf - 2;
  g.gfb = g.Tb / kR;
  g.NGb = (2 * p.Lf) / kR - g.gfb + 1;
  g.Tc = p.Lf + p.sc - 2;
  g.gfc = g.Tc / kR;
  g.NGc = (2 * p.Lf) / kR - g.gfc + 1;
  g.NCX = kR * (g.NGb + 2);
  return g;
}

// Shared-memory carve-up (identical on host and device).
struct Layout {
  int rw;                 // words per staged row
  int n_stage_rows;       // kc * (nlv + nrv)
  int n_const_rows;       // D + D*D + NT
  int n_units;            // partial-sum units
  size_t off_stage, off_sinfo, off_const, off_cinfo, off_cur, off_curinfo, off_s, off_sinf,
      off_u, off_uinf, off_ct, off_ctinf, off_part, off_col, off_uout, off_flag, total;
};

__host__ __device__ inline Layout make_layout(const Params& p) {
  Geo g = make_geo(p);
  Layout L;
  L.rw = row_words(p.RS);
  L.n_stage_rows = p.kc * (p.nlv + p.nrv);
  L.n_const_rows = p.D + p.D * p.D + p.NT;
  int ns = p.nthreads / ((p.NP > 0 ? p.NP : 1) * ((g.NGb + 1) / 2));
  if (ns < 1) ns = 1;
  int units_a = ns * (p.NP > 0 ? p.NP : 1);
  int units_b = p.D * p.D + p.NT;  // numerator items
  int units_c = p.D;
  int u = units_a;
  if (units_b > u) u = units_b;
  if (units_c > u) u = units_c;
  L.n_units = u;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o += (bytes + 15) / 16 * 16;
    return r;
  };
  L.off_stage = take(sizeof(int32_t) * (size_t)L.n_stage_rows * L.rw);
  L.off_sinfo = take(sizeof(int2) * (size_t)L.n_stage_rows);
  L.off_const = take(sizeof(int32_t) * (size_t)L.n_const_rows * L.rw);
  L.off_cinfo = take(sizeof(int2) * (size_t)L.n_const_rows);
  L.off_cur = take(sizeof(int32_t) * (size_t)p.D * L.rw);
  L.off_curinfo = take(sizeof(int2) * (size_t)p.D);
  L.off_s = take(sizeof(int32_t) * (size_t)(p.NP > 0 ? p.NP : 1) * L.rw);
  L.off_sinf = take(sizeof(int2) * (size_t)(p.NP > 0 ? p.NP : 1));
  L.off_u = take(sizeof(int32_t) * (size_t)p.D * L.rw);
  L.off_uinf = take(sizeof(int2) * (size_t)p.D);
  L.off_ct = take(sizeof(int32_t) * (size_t)L.rw);
  L.off_ctinf = take(sizeof(int2));
  L.off_part = take(sizeof(int64_t) * (size_t)L.n_units * part_stride(g.NCX));
  L.off_col = take(sizeof(int64_t) * (size_t)(p.NP + p.D) * g.NCX);  // V_p then U_m
  L.off_uout = take(sizeof(int) * (size_t)L.n_units);
  L.off_flag = take(sizeof(int) * 4);
  L.total = o;
  return L;
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ void copy_row(int32_t* dst, const int32_t* __restrict__ src, int RS) {
  for (int d = threadIdx.x; d < RS; d += blockDim.x) dst[d] = src[d];
}

// MB = CTAs resident per SM the register budget is sized for (1: 255 regs;
// 2: 128 regs -- ensembles, where several trajectories per SM hide the
// per-order barrier and HBM latencies of one another).
// MB = 4: 128-thread CTAs at 128 registers, four trajectories per SM (small K).
template <int NPT, int MB>
__global__ void __launch_bounds__(MB >= 8 ? 64 : MB >= 4 ? 128 : 256, MB) taylor_team_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Geo g = make_geo(p);
  const Layout L = make_layout(p);
  const int tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, nwarps = nt >> 5;
  const int traj = blockIdx.x;
  if (traj >= p.n_traj) return;

  int32_t* stage = (int32_t*)(smem + L.off_stage);
  int2* stinfo = (int2*)(smem + L.off_sinfo);
  int32_t* crow = (int32_t*)(smem + L.off_const);
  int2* cinfo = (int2*)(smem + L.off_cinfo);
  int32_t* cur = (int32_t*)(smem + L.off_cur);
  int2* curinfo = (int2*)(smem + L.off_curinfo);
  int32_t* srow = (int32_t*)(smem + L.off_s);
  int2* sinf = (int2*)(smem + L.off_sinf);
  int32_t* urow = (int32_t*)(smem + L.off_u);
  int2* uinf = (int2*)(smem + L.off_uinf);
  int32_t* ctrow = (int32_t*)(smem + L.off_ct);
  int2* ctinf = (int2*)(smem + L.off_ctinf);
  int64_t* part = (int64_t*)(smem + L.off_part);
  int64_t* colsum = (int64_t*)(smem + L.off_col);
  int* uout = (int*)(smem + L.off_uout);
  int* flag = (int*)(smem + L.off_flag);
  const int rw = L.rw;
  auto ROW = [&](int32_t* base, int r) { return base + (size_t)r * rw + kPad; };

  // zero all of shared memory once (pads stay zero forever)
  for (size_t w = tid; w < L.total / 4; w += nt) ((int32_t*)smem)[w] = 0;
  if (tid == 0) flag[0] = 0;
  __syncthreads();

  // constant rows: cst (D), lin (D*D), q (NT)
  for (int r = 0; r < L.n_const_rows; r++) {
    const int32_t* src = r < p.D ? p.cst + (size_t)r * p.RS
                         : r < p.D + p.D * p.D ? p.lin + (size_t)(r - p.D) * p.RS
                                                : p.q + (size_t)(r - p.D - p.D * p.D) * p.RS;
    copy_row(ROW(crow, r), src, p.RS);
  }
  __syncthreads();
  for (int r = warp; r < L.n_const_rows; r += nwarps) {
    int bot = 1 << 30, tp = -1;
    const int32_t* row = ROW(crow, r);
    for (int d = (tid & 31); d < p.W; d += 32)
      if (row[d]) {
        bot = min(bot, d);
        tp = max(tp, d);
      }
    bot = __reduce_min_sync(0xffffffffu, bot);
    tp = __reduce_max_sync(0xffffffffu, tp);
    if ((tid & 31) == 0) cinfo[r] = make_int2(tp >= 0 ? bot : p.W, tp);
  }

  const size_t traj_rows = (size_t)p.D * (p.N + 1);
  int32_t* gcoef = p.coef + (size_t)traj * traj_rows * p.RS;
  int2* ginfo = p.rinfo + (size_t)traj * traj_rows;
  int32_t* gstate = p.state + (size_t)traj * p.D * p.RS;
  auto GROW = [&](int m, int i) { return gcoef + ((size_t)m * (p.N + 1) + i) * p.RS; };
  auto GINF = [&](int m, int i) -> int2& { return ginfo[(size_t)m * (p.N + 1) + i]; };

  // initial state -> cur rows (normalised info computed from digits)
  for (int m = 0; m < p.D; m++) copy_row(ROW(cur, m), gstate + (size_t)m * p.RS, p.RS);
  __syncthreads();

  // phase A units: (k slot, pair, group pair) -- see team_units()
  const int NGh = (g.NGb + 1) / 2;
  const int unit_per_slot = max(1, p.NP) * NGh;
  const int ns_a = max(1, nt / unit_per_slot);  // k slots in phase A
  int status = 0;
  MacCount mcount;
  MacCount* mc = p.counters ? &mcount : nullptr;

  for (int n = p.start_step + 1; n <= p.n_steps; n++) {
    // coefficient row 0 = state
    for (int m = warp; m < p.D; m += nwarps) {
      int bot = 1 << 30, tp = -1;
      const int32_t* row = ROW(cur, m);
      for (int d = (tid & 31); d < p.W; d += 32)
        if (row[d]) {
          bot = min(bot, d);
          tp = max(tp, d);
        }
      bot = __reduce_min_sync(0xffffffffu, bot);
      tp = __reduce_max_sync(0xffffffffu, tp);
      if ((tid & 31) == 0) {
        curinfo[m] = make_int2(tp >= 0 ? bot : p.W, tp);
        GINF(m, 0) = curinfo[m];
      }
    }
    for (int m = 0; m < p.D; m++)
      for (int d = tid; d < p.RS; d += nt) GROW(m, 0)[d] = ROW(cur, m)[d];
    __syncthreads();

    for (int i = 0; i < p.N; i++) {
      // ===================== phase A: Cauchy sums =====================
      if (p.NP > 0) {
        // unit = (slot, pair q, group pair h): the thread accumulates column
        // windows h and NGb-1-h of pair q. Low windows hold ~W digit products
        // per column, high ones few; pairing them gives every lane the same
        // work (a warp runs at its slowest lane).
        const int slot = tid / unit_per_slot, rem = tid % unit_per_slot;
        const int q = rem / NGh, h = rem % NGh;
        const bool active = slot < ns_a;
        const int gB = g.NGb - 1 - h;
        const bool twoB = gB != h;
        const int c0A = kR * (g.gfb + h), c0B = kR * (g.gfb + gB);
        Acc accA, accB;
        acc_zero(accA);
        acc_zero(accB);
        int cntA = 0, cntB = 0;
        const int nrows = p.nlv + p.nrv;
        for (int k0 = 0; k0 <= i; k0 += p.kc) {
          const int kcn = min(p.kc, i + 1 - k0);
          // stage rows: one flat, 16-byte vectorised copy of all kcn*nrows rows
          {
            const int q4 = p.RS / 4;
            const int total = kcn * nrows * q4;
            for (int e = tid; e < total; e += nt) {
              const int r = e / q4, w = e - r * q4;
              const int kk = r / nrows, v = r - kk * nrows;
              const int k = k0 + kk;
              const int32_t* src = v < p.nlv ? GROW(p.lvar[v], i - k) : GROW(p.rvar[v - p.nlv], k);
              const int4 v4 = __ldcg(reinterpret_cast<const int4*>(src) + w);
              int32_t* dst = ROW(stage, r) + 4 * w;
              dst[0] = v4.x;
              dst[1] = v4.y;
              dst[2] = v4.z;
              dst[3] = v4.w;
            }
            for (int r = tid; r < kcn * nrows; r += nt) {
              const int kk = r / nrows, v = r - kk * nrows;
              const int k = k0 + kk;
              stinfo[r] = v < p.nlv ? GINF(p.lvar[v], i - k) : GINF(p.rvar[v - p.nlv], k);
            }
          }
          __syncthreads();
          if (active) {
            for (int kk = slot; kk < kcn; kk += ns_a) {
              const int ra = kk * nrows + p.pl[q];
              const int rb = kk * nrows + p.nlv + p.pr[q];
              mac_group(accA, cntA, ROW(stage, ra), stinfo[ra], ROW(stage, rb), stinfo[rb], c0A, g.Tb, mc);
              if (twoB)
                mac_group(accB, cntB, ROW(stage, ra), stinfo[ra], ROW(stage, rb), stinfo[rb], c0B, g.Tb, mc);
            }
          }
          __syncthreads();
        }
        // partials: unit = slot * NP + q, columns relative to Tb
        const int pst = part_stride(g.NCX);
        if (active) {
          int64_t* pr = part + (size_t)(slot * p.NP + q) * pst;
          acc_fold(accA, c0A, g.Tb);
#pragma unroll
          for (int r = 0; r < kR; r++) {
            int c = c0A + r - g.Tb;
            if (c >= 0) pr[part_idx(c)] = accA.v[r];
          }
          if (twoB) {
            acc_fold(accB, c0B, g.Tb);
#pragma unroll
            for (int r = 0; r < kR; r++) {
              int c = c0B + r - g.Tb;
              if (c >= 0) pr[part_idx(c)] = accB.v[r];
            }
          }
        }
        for (int u = tid; u < ns_a * p.NP; u += nt) uout[u] = u % p.NP;
        __syncthreads();
        if (active) {
          int64_t* pr = part + (size_t)(slot * p.NP + q) * pst;
          pr[part_idx(c0A + kR - g.Tb)] += accA.v[kR];  // carries land in distinct columns (h+1 <= NGb-h)
          if (twoB) pr[part_idx(c0B + kR - g.Tb)] += accB.v[kR];
        }
        __syncthreads();
        // reduce units -> colsum[q][c]
        const int ncol = kR * (g.gfb + g.NGb) - g.Tb + 1;
        for (int e = tid; e < p.NP * ncol; e += nt) {
          int q = e / ncol, c = e % ncol;
          int64_t s = 0;
          for (int sl = 0; sl < ns_a; sl++) s += part[(size_t)(sl * p.NP + q) * pst + part_idx(c)];
          colsum[(size_t)q * g.NCX + c] = s;
        }
        // clear partials for the next use
        __syncthreads();
        for (size_t w = tid; w < (size_t)ns_a * p.NP * pst; w += nt) part[w] = 0;
        for (int q = warp; q < p.NP; q += nwarps) {
          if (!p.pair_round[q]) continue;
          bool o = warp_normalize(colsum + (size_t)q * g.NCX, ncol, 2, p.W, ROW(srow, q), &sinf[q], 0);
          if (o && (tid & 31) == 0) flag[0] = 1;
        }
        __syncthreads();
      }
      // ===================== phase B: numerators =====================
      {
        // product items: non-small-integer linear coefficients and non-small-integer q terms
        const int nlin = p.D * p.D;
        const int nitems = nlin + p.NT;
        for (int u = tid; u < nitems; u += nt) uout[u] = u < nlin ? u / p.D : p.teq[u - nlin];
        for (int e = tid; e < nitems * g.NGb; e += nt) {
          const int it = e / g.NGb, grp = e % g.NGb;
          const int c0 = kR * (g.gfb + grp);
          const int32_t *A, *B;
          int2 ia, ib;
          if (it < nlin) {
            if (p.lin_small[it]) continue;
            const int m = it / p.D, j = it % p.D;
            A = ROW(crow, p.D + m * p.D + j);
            ia = cinfo[p.D + m * p.D + j];
            B = ROW(cur, j);
            ib = curinfo[j];
          } else {
            const int t = it - nlin;
            if (p.tq_small[t]) continue;
            A = ROW(crow, p.D + nlin + t);
            ia = cinfo[p.D + nlin + t];
            B = ROW(srow, p.tpair[t]);
            ib = sinf[p.tpair[t]];
          }
          Acc acc;
          acc_zero(acc);
          int cnt = 0;
          mac_group(acc, cnt, A, ia, B, ib, c0, g.Tb, mc);
          acc_fold(acc, c0, g.Tb);
          int64_t* pr = part + (size_t)it * g.NCX;
#pragma unroll
          for (int r = 0; r <= kR; r++) {
            int c = c0 + r - g.Tb;
            if (c >= 0) atomicAdd((unsigned long long*)&pr[c], (unsigned long long)acc.v[r]);
          }
        }
        __syncthreads();
        const int ncol = kR * (g.gfb + g.NGb) - g.Tb + 1;
        int64_t* ucol = colsum + (size_t)p.NP * g.NCX;
        for (int e = tid; e < p.D * ncol; e += nt) {
          const int m = e / ncol, c = e % ncol;
          int64_t s = 0;
          for (int u = 0; u < nitems; u++)
            if (uout[u] == m) s += part[(size_t)u * g.NCX + c];
          if (c >= 2 && c - 2 < p.W) {
            const int dgt = c - 2;
            if (i == 0) s += ROW(crow, m)[dgt];
            for (int j = 0; j < p.D; j++)
              if (p.lin_small[m * p.D + j]) s += (int64_t)p.lin_int[m * p.D + j] * ROW(cur, j)[dgt];
          }
          for (int t = 0; t < p.NT; t++)
            if (p.teq[t] == m && p.tq_small[t]) s += (int64_t)p.tq_int[t] * colsum[(size_t)p.tpair[t] * g.NCX + c];
          ucol[(size_t)m * g.NCX + c] = s;
        }
        __syncthreads();
        for (size_t w = tid; w < (size_t)nitems * g.NCX; w += nt) part[w] = 0;
        // tau/(i+1) row for phase C: staged (with its digit range) by a warp
        // that has no normalisation to do, in the same barrier phase
        const int ctw = p.D < nwarps ? p.D : -1;
        if (ctw < 0) copy_row(ROW(ctrow, 0), p.ctab + (size_t)i * p.RS, p.RS);
        for (int m = warp; m < p.D; m += nwarps) {
          bool o = warp_normalize(ucol + (size_t)m * g.NCX, ncol, 2, p.W, ROW(urow, m), &uinf[m], 0);
          if (o && (tid & 31) == 0) flag[0] = 1;
        }
        if (warp == ctw) {
          int bot = 1 << 30, tp = -1;
          int32_t* row = ROW(ctrow, 0);
          const int32_t* src = p.ctab + (size_t)i * p.RS;
          for (int d = (tid & 31); d < p.RS; d += 32) {
            const int32_t v = src[d];
            row[d] = v;
            if (d < p.W && v) {
              bot = min(bot, d);
              tp = max(tp, d);
            }
          }
          bot = __reduce_min_sync(0xffffffffu, bot);
          tp = __reduce_max_sync(0xffffffffu, tp);
          if ((tid & 31) == 0) ctinf[0] = make_int2(tp >= 0 ? bot : p.W, tp);
        }
        __syncthreads();
        if (ctw < 0) {
          if (warp == 0) {
            int bot = 1 << 30, tp = -1;
            const int32_t* row = ROW(ctrow, 0);
            for (int d = (tid & 31); d < p.W; d += 32)
              if (row[d]) {
                bot = min(bot, d);
                tp = max(tp, d);
              }
            bot = __reduce_min_sync(0xffffffffu, bot);
            tp = __reduce_max_sync(0xffffffffu, tp);
            if (tid == 0) ctinf[0] = make_int2(tp >= 0 ? bot : p.W, tp);
          }
          __syncthreads();
        }
      }
      // ===================== phase C: scale by tau/(i+1) =====================
      {
        for (int e = tid; e < p.D * g.NGc; e += nt) {
          const int m = e / g.NGc, grp = e % g.NGc;
          const int c0 = kR * (g.gfc + grp);
          Acc acc;
          acc_zero(acc);
          int cnt = 0;
          mac_group(acc, cnt, ROW(urow, m), uinf[m], ROW(ctrow, 0), ctinf[0], c0, g.Tc, mc);
          acc_fold(acc, c0, g.Tc);
          int64_t* pr = part + (size_t)m * g.NCX;
#pragma unroll
          for (int r = 0; r <= kR; r++) {
            int c = c0 + r - g.Tc;
            if (c >= 0) atomicAdd((unsigned long long*)&pr[c], (unsigned long long)acc.v[r]);
          }
        }
        __syncthreads();
        const int ncol = kR * (g.gfc + g.NGc) - g.Tc + 1;
        for (int m = warp; m < p.D; m += nwarps) {
          bool o = warp_normalize(part + (size_t)m * g.NCX, ncol, 2, p.W, ROW(cur, m), &curinfo[m], 0);
          if (o && (tid & 31) == 0) flag[0] = 1;
        }
        __syncthreads();
        for (size_t w = tid; w < (size_t)p.D * g.NCX; w += nt) part[w] = 0;
        for (int m = 0; m < p.D; m++)
          for (int d = tid; d < p.RS; d += nt) GROW(m, i + 1)[d] = ROW(cur, m)[d];
        if (tid < p.D) GINF(tid, i + 1) = curinfo[tid];
        __syncthreads();
      }
    }
    // ===================== state update: exact sum of rows, round to P bits ===========
    {
      const int ncol = p.W + 3;
      for (int e = tid; e < p.D * ncol; e += nt) {
        int m = e / ncol, c = e % ncol;
        int64_t s = 0;
        if (c < p.W)
          for (int i = 0; i <= p.N; i++) s += GROW(m, i)[c];
        colsum[(size_t)m * g.NCX + c] = s;
      }
      __syncthreads();
      for (int m = warp; m < p.D; m += nwarps) {
        bool o = warp_normalize(colsum + (size_t)m * g.NCX, ncol, 0, p.W, ROW(cur, m), &curinfo[m], p.P);
        if (o && (tid & 31) == 0) flag[0] = 1;
      }
      __syncthreads();
      // record
      const bool rec = (n % p.stride == 0) || (n == p.n_steps);
      if (rec) {
        int slot = (n % p.stride == 0) ? (n / p.stride - p.start_step / p.stride)
                                       : (p.n_steps / p.stride - p.start_step / p.stride + 1);
        int32_t* dst = p.rec + ((size_t)slot * p.n_traj + traj) * p.D * p.RS;
        for (int m = 0; m < p.D; m++)
          for (int d = tid; d < p.RS; d += nt) dst[(size_t)m * p.RS + d] = ROW(cur, m)[d];
      }
      __syncthreads();
    }
  }
  for (int m = 0; m < p.D; m++)
    for (int d = tid; d < p.RS; d += nt) gstate[(size_t)m * p.RS + d] = ROW(cur, m)[d];
  if (tid == 0) {
    status = flag[0] ? kOverflow : kOk;
    p.status[traj] = status;
  }
  if (mc) {
    atomicAdd(&p.counters[0], mcount.useful);
    atomicAdd(&p.counters[1], mcount.executed);
  }
}

// Integer-pipe roofline probe: every thread runs 8 independent IMAD.WIDE
// chains (s64 += s32 * s32) -- the instruction the Cauchy loop is built on.
__global__ void __launch_bounds__(512) imad_wide_probe(int iters, int32_t seed, long long* out) {
  int64_t acc[8];
#pragma unroll
  for (int c = 0; c < 8; c++) acc[c] = seed + c;
  int32_t x = threadIdx.x | 1, y = blockIdx.x | 3;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 8; u++) {
#pragma unroll
      for (int c = 0; c < 8; c++) {
        int64_t d;  // one fused IMAD.WIDE (s64 += s32 * s32), as in the kernels' inner loops
        asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(x + c), "r"(y), "l"(acc[c]));
        acc[c] = d;
      }
      y += u;
    }
  }
  int64_t s = 0;
#pragma unroll
  for (int c = 0; c < 8; c++) s ^= acc[c];
  if (s == 0x123456789LL) out[0] = s;
}

cudaError_t launch_imad_probe(int blocks, int threads, int iters, long long* out, cudaStream_t s) {
  imad_wide_probe<<<blocks, threads, 0, s>>>(iters, 7, out);
  return cudaGetLastError();
}

cudaError_t launch_team_kernel(const Params& p, size_t smem, cudaStream_t stream) {
  const int npt = p.NP <= 1 ? 1 : p.NP <= 2 ? 2 : p.NP <= 4 ? 4 : 8;
  const bool two = p.team_mb >= 2 && npt <= 2, four = p.team_mb >= 4 && npt <= 2, eight = p.team_mb >= 8 && npt <= 2;
  const void* fn = npt == 1   ? (eight ? (const void*)taylor_team_kernel<1, 8>
                                 : four ? (const void*)taylor_team_kernel<1, 4>
                                 : two ? (const void*)taylor_team_kernel<1, 2>
                                       : (const void*)taylor_team_kernel<1, 1>)
                   : npt == 2 ? (eight ? (const void*)taylor_team_kernel<2, 8>
                                 : four ? (const void*)taylor_team_kernel<2, 4>
                                 : two ? (const void*)taylor_team_kernel<2, 2>
                                       : (const void*)taylor_team_kernel<2, 1>)
                   : npt == 4 ? (const void*)taylor_team_kernel<4, 1>
                              : (const void*)taylor_team_kernel<8, 1>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  Params pc = p;
  void* args[] = {&pc};
  return cudaLaunchKernel(fn, dim3(p.n_traj), dim3(p.nthreads), args, smem, stream);
}

size_t smem_bytes(const Params& p) { return make_layout(p).total; }

}  // namespace mpt
