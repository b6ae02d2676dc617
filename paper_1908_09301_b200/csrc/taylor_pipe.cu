// Warp-specialised, pipelined Taylor kernel for one trajectory per thread-
// block cluster (G = 1..16 CTAs on G SMs), coefficient rows resident in shared
// memory. This is the latency-optimised path for the single-trajectory
// configurations.
//
// The Cauchy sum of order i is split into the part that needs the newest
// coefficient and a lookahead part that does not:
//
//     S_p(i) = a_i b_0 + a_0 b_i  +  P_p(i),   P_p(i) = sum_{k=1}^{i-1} a_{i-k} b_k
//
// P_p(i+1) only involves coefficients 1..i, so it is computed by the BULK
// warps of every CTA (k = rank (mod G)) while the CHAIN warps finish order i:
//
//   chain warps  C1  new-term products a_i b_0, a_0 b_i and non-integer
//                    linear products (product slots in smem)
//                C2  warp m: U_m = sum q_t (P_p(i) + new terms) + linear + c_m,
//                    normalise (warp-level, no CTA barrier)
//                C3  warp m: coef_m[i+1] = rnd(U_m (x) tau/(i+1)), publish row
//   bulk warps   P_p(i+1) partial columns -> pushed with st.shared::cluster
//                into slot [rank] of every CTA's receive buffer (parity i+1)
//   ---- one cluster barrier per order (arrive.release / wait.acquire)
//
// Per-order latency is max(chain, bulk) plus one cluster barrier instead of a
// chain of CTA-wide phases. Arithmetic is identical to oracle/fixmodel.c
// (column sums are exact integers, so the split does not change any bit).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "mpt_common.cuh"
#include "mpt_device.cuh"

namespace cg = cooperative_groups;

namespace mpt {
namespace pipe {

constexpr int kChainWarps = 4;  // >= D; warp m < D owns equation m
constexpr int kBulkWarps = 8;
constexpr int kThreads = 32 * (kChainWarps + kBulkWarps);
constexpr int kMaxChainProducts = 2 * kMaxP + kMaxD * kMaxD;
constexpr int kPch = 3;  // p-range chunks per column group in warp products
constexpr int kMaxG = 16;

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
  int rs, nslots, base[kMaxD], full[kMaxD], ncrow;
  int nbu;  // bulk units (slots * NP)
  size_t off_rows, off_rinfo, off_crow, off_cinfo, off_recv, off_bpart, off_bpcar, off_bcol, off_prod, off_wsc,
      off_wcar, off_ucol, off_ssum, off_flag, total;
};

// crow rows: cst D | lin D*D | q NT | ctab x2 | U D | CUR x2 (D each) | ZERO D
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
  L.ncrow = p.D + p.D * p.D + p.NT + 2 + p.D + 2 * p.D + p.D;
  const Geo g = make_geo(p);
  const int ns = (32 * kBulkWarps) / g.NGb;
  L.nbu = ns * (p.NP > 0 ? p.NP : 1);
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
  L.off_recv = take(sizeof(int64_t) * 2 * (size_t)G * (p.NP > 0 ? p.NP : 1) * g.ncolb);
  L.off_bpart = take(sizeof(uint32_t) * (size_t)L.nbu * g.NCX);
  L.off_bpcar = take(sizeof(int64_t) * (size_t)L.nbu * g.NGb);
  L.off_bcol = take(sizeof(int64_t) * (size_t)(p.NP > 0 ? p.NP : 1) * g.ncolb);
  L.off_prod = take(sizeof(int64_t) * (size_t)kMaxChainProducts * g.NCX);
  L.off_wsc = take(sizeof(uint32_t) * (size_t)kChainWarps * kPch * g.NCX);
  L.off_wcar = take(sizeof(int64_t) * (size_t)kChainWarps * kPch * (g.NGb + 1));
  L.off_ucol = take(sizeof(int64_t) * (size_t)kChainWarps * g.NCX);
  L.off_ssum = take(sizeof(int64_t) * (size_t)p.D * (p.W + 3));
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

// sum_c of the folded (digit, carry) units: digits of the group owning c and
// the carry of the group below it
__device__ __forceinline__ int64_t unit_col(const uint32_t* part, const int64_t* pcar, int u0, int ustride, int n,
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

// One warp computes the truncated product A (x) B into columns out[0..ncol)
// (relative to T): lanes = (column group, p-chunk), partials through a
// warp-private scratch, then one column sum per lane. `acc_into` adds.
__device__ __forceinline__ void warp_product(const int32_t* A, int2 ia, const int32_t* B, int2 ib, int T, int gf,
                                             int ng, int ncol, int ncx, uint32_t* wsc, int64_t* wcar, int64_t* out,
                                             bool acc_into, MacCount* mc) {
  const int lane = threadIdx.x & 31;
  for (int e = lane; e < ng * kPch; e += 32) {
    const int grp = e / kPch, pc = e - grp * kPch;
    const int c0 = kR * (gf + grp);
    Acc acc;
    acc_zero(acc);
    int2 ja = ia;
    const int plo = max(ia.x, c0 - ib.y), phi = min(ia.y, c0 + kR - 1 - ib.x);
    if (plo <= phi) {
      const int b0 = plo / kR, nb = phi / kR - b0 + 1;
      const int per = (nb + kPch - 1) / kPch;
      const int blo = b0 + pc * per, bhi = min(b0 + nb, blo + per) - 1;
      if (blo <= bhi) {
        ja.x = max(ia.x, blo * kR);
        ja.y = min(ia.y, bhi * kR + kR - 1);
        int cnt = 0;
        mac_group(acc, cnt, A, ja, B, ib, c0, T, mc);
        acc_fold(acc, c0, T);
      }
    }
    uint32_t* part = wsc + (size_t)pc * ncx;
#pragma unroll
    for (int r = 0; r < kR; r++) {
      const int c = c0 + r - T;
      if (c >= 0) part[c] = (uint32_t)acc.v[r];
    }
    wcar[(size_t)pc * (ng + 1) + grp] = acc.v[kR];
  }
  __syncwarp();
  for (int c = lane; c < ncol; c += 32) {
    const int64_t s = unit_col(wsc, wcar, 0, 1, kPch, ncx, ng + 1, c, T, gf, ng);
    out[c] = acc_into ? out[c] + s : s;
  }
  __syncwarp();
}

template <int NPT>
__global__ void __launch_bounds__(kThreads, 1) taylor_pipe_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(16) unsigned char smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int G = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int traj = blockIdx.x / G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool is_chain = warp < kChainWarps;
  const Geo g = make_geo(p);
  const Layout L = make_layout(p, G);
  const int NPp = p.NP > 0 ? p.NP : 1;

  int32_t* rows = (int32_t*)(smem + L.off_rows) + kPad;
  int2* rinfo = (int2*)(smem + L.off_rinfo);
  int32_t* crow = (int32_t*)(smem + L.off_crow) + kPad;
  int2* cinfo = (int2*)(smem + L.off_cinfo);
  int64_t* recv = (int64_t*)(smem + L.off_recv);
  uint32_t* bpart = (uint32_t*)(smem + L.off_bpart);
  int64_t* bpcar = (int64_t*)(smem + L.off_bpcar);
  int64_t* bcol = (int64_t*)(smem + L.off_bcol);
  int64_t* prod = (int64_t*)(smem + L.off_prod);
  uint32_t* wsc = (uint32_t*)(smem + L.off_wsc);
  int64_t* wcar = (int64_t*)(smem + L.off_wcar);
  int64_t* ucol = (int64_t*)(smem + L.off_ucol);
  int64_t* ssum = (int64_t*)(smem + L.off_ssum);
  int* flag = (int*)(smem + L.off_flag);
  const int rs = L.rs;
  const int CR_CST = 0, CR_LIN = p.D, CR_Q = CR_LIN + p.D * p.D, CR_CT = CR_Q + p.NT, CR_U = CR_CT + 2,
            CR_CUR = CR_U + p.D, CR_ZERO = CR_CUR + 2 * p.D;
  auto CROW = [&](int r) { return crow + (size_t)r * rs; };
  __shared__ int s_base[kMaxD], s_full[kMaxD];
  __shared__ int64_t* s_recv_remote[kMaxG];
  // chain product list of the current order (rebuilt per order by warp 0)
  __shared__ int s_np, s_pa[kMaxChainProducts], s_pb[kMaxChainProducts], s_ptg[kMaxChainProducts];
  if (tid < kMaxD) {
    s_base[tid] = tid < p.D ? L.base[tid] : 0;
    s_full[tid] = tid < p.D ? L.full[tid] : 1;
  }
  if (tid < kMaxG) s_recv_remote[tid] = tid < G ? cluster.map_shared_rank(recv, tid) : nullptr;
  auto has_row = [&](int v, int k) { return s_full[v] || (k % G) == rank; };
  auto SLOT = [&](int v, int k) { return s_base[v] + (s_full[v] ? k : k / G); };
  auto ROW = [&](int v, int k) { return rows + (size_t)SLOT(v, k) * rs; };
  const size_t recv_par = (size_t)G * NPp * g.ncolb;  // int64 per parity

  for (size_t w = tid; w < L.total / 4; w += kThreads) ((int32_t*)smem)[w] = 0;
  __syncthreads();
  for (int r = 0; r < CR_CT; r++) {
    const int32_t* src = r < CR_LIN ? p.cst + (size_t)r * p.RS
                         : r < CR_Q ? p.lin + (size_t)(r - CR_LIN) * p.RS
                                    : p.q + (size_t)(r - CR_Q) * p.RS;
    for (int d = tid; d < p.W; d += kThreads) CROW(r)[d] = src[d];
  }
  int32_t* gstate = p.state + (size_t)traj * p.D * p.RS;
  for (int m = 0; m < p.D; m++)
    for (int d = tid; d < p.W; d += kThreads) CROW(CR_ZERO + m)[d] = gstate[(size_t)m * p.RS + d];
  __syncthreads();
  for (int r = warp; r < CR_CT; r += kThreads / 32) {
    int2 inf = row_info_warp(CROW(r), p.W);
    if (lane == 0) cinfo[r] = inf;
  }
  MacCount mcount;
  MacCount* mc = p.counters ? &mcount : nullptr;
  const int nlin = p.D * p.D;
  cluster.sync();  // remote receive buffers exist and are zero

  for (int n = p.start_step + 1; n <= p.n_steps; n++) {
    // ---- order 0 of this step: coefficient row 0 = state (ZERO rows) -------------
    if (is_chain) {
      for (int m = warp; m < p.D; m += kChainWarps) {
        const int32_t* z = CROW(CR_ZERO + m);
        const int2 inf = row_info_warp(z, p.W);
        for (int d = lane; d < p.W + 3; d += 32) {
          const int32_t v = d < p.W ? z[d] : 0;
          ssum[(size_t)m * (p.W + 3) + d] = v;
          if (d < p.W) {
            CROW(CR_CUR + m)[d] = v;  // CUR parity 0 = coefficient 0
            if (has_row(m, 0)) ROW(m, 0)[d] = v;
          }
        }
        if (lane == 0) {
          cinfo[CR_ZERO + m] = inf;
          cinfo[CR_CUR + m] = inf;
          if (has_row(m, 0)) rinfo[SLOT(m, 0)] = inf;
        }
      }
      // tau/(0+1) row into ctab buffer 0
      for (int d = tid; d < p.W; d += 32 * kChainWarps) CROW(CR_CT)[d] = __ldg(p.ctab + d);
    }
    __syncthreads();

    for (int i = 0; i < p.N; i++) {
      const int par = i & 1;
      const bool tlog = p.dbg && n == p.start_step + 1 && rank == 0 && i < 200 && lane == 0;
#define TSTAMP(ev) \
  if (tlog) p.dbg[(size_t)i * 16 + (ev)] = (long long)clock64();
      if (warp == 0) TSTAMP(0);
      if (is_chain) {
        // ================= chain ================================================
        const int32_t* cur = CROW(CR_CUR + par * p.D);  // coefficient i, variable 0
        const int2* curinf = cinfo + CR_CUR + par * p.D;
        if (tid == 0) {
          int np = 0;
          for (int q = 0; q < p.NP; q++) {
            // new terms of pair q: k = 0 (a_i b_0) and k = i (a_0 b_i)
            s_pa[np] = q * 4 + 0;  // encoded below
            s_ptg[np] = q;
            np++;
            if (i > 0) {
              s_pa[np] = q * 4 + 1;
              s_ptg[np] = q;
              np++;
            }
          }
          for (int it = 0; it < nlin; it++)
            if (!p.lin_small[it] && cinfo[CR_LIN + it].y >= 0) {
              s_pa[np] = -1 - it;
              s_ptg[np] = NPp + it / p.D;
              np++;
            }
          s_np = np;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(32 * kChainWarps));
        if (warp == 0) TSTAMP(1);
        // C1: chain products, one warp per product
        const int npr = s_np;
        for (int pr = warp; pr < npr; pr += kChainWarps) {
          const int code = s_pa[pr];
          const int32_t *A, *B;
          int2 ia, ib;
          if (code >= 0) {
            const int q = code >> 2, which = code & 3;
            const int va = p.pj[q], vb = p.pk[q];
            if (which == 0) {  // a_i b_0
              A = cur + (size_t)va * rs;
              ia = curinf[va];
              B = CROW(CR_ZERO + vb);
              ib = cinfo[CR_ZERO + vb];
            } else {  // a_0 b_i
              A = CROW(CR_ZERO + va);
              ia = cinfo[CR_ZERO + va];
              B = cur + (size_t)vb * rs;
              ib = curinf[vb];
            }
          } else {
            const int it = -1 - code, j = it % p.D;
            A = CROW(CR_LIN + it);
            ia = cinfo[CR_LIN + it];
            B = cur + (size_t)j * rs;
            ib = curinf[j];
          }
          warp_product(A, ia, B, ib, g.Tb, g.gfb, g.NGb, g.ncolb, g.NCX, wsc + (size_t)warp * kPch * g.NCX,
                       wcar + (size_t)warp * kPch * (g.NGb + 1), prod + (size_t)pr * g.NCX, false, mc);
        }
        asm volatile("bar.sync 1, %0;" ::"r"(32 * kChainWarps));
        if (warp == 0) TSTAMP(2);
        // C2 + C3: warp m owns equation m
        for (int m = warp; m < p.D; m += kChainWarps) {
          int64_t* uc = ucol + (size_t)warp * g.NCX;
          const int64_t* rv = recv + (size_t)par * recv_par;
          for (int c = lane; c < g.ncolb; c += 32) {
            int64_t s = 0;
            for (int t = 0; t < p.NT; t++) {
              if (p.teq[t] != m) continue;
              const int q = p.tpair[t];
              int64_t v = 0;
              if (i >= 2) {  // lookahead part P_q(i) from every CTA's bulk warps
#pragma unroll 4
                for (int r = 0; r < G; r++) v += rv[((size_t)r * NPp + q) * g.ncolb + c];
              }
              for (int pr = 0; pr < npr; pr++)
                if (s_ptg[pr] == q) v += prod[(size_t)pr * g.NCX + c];
              s += (int64_t)p.tq_int[t] * v;
            }
            for (int pr = 0; pr < npr; pr++)
              if (s_ptg[pr] == NPp + m) s += prod[(size_t)pr * g.NCX + c];
            if (c >= 2 && c - 2 < p.W) {
              const int dgt = c - 2;
              if (i == 0) s += CROW(CR_CST + m)[dgt];
              for (int j = 0; j < p.D; j++)
                if (p.lin_small[m * p.D + j]) s += (int64_t)p.lin_int[m * p.D + j] * cur[(size_t)j * rs + dgt];
            }
            uc[c] = s;
          }
          __syncwarp();
          if (warp == 2) TSTAMP(3);
          if (warp_normalize_small(uc, g.ncolb, 2, p.W, CROW(CR_U + m), &cinfo[CR_U + m], 0) && lane == 0) flag[0] = 1;
          if (warp == 2) TSTAMP(4);
          // C3: scale by tau/(i+1)
          const int32_t* ct = CROW(CR_CT + par);
          const int2 ctinf = row_info_warp(ct, p.W);
          warp_product(CROW(CR_U + m), cinfo[CR_U + m], ct, ctinf, g.Tc, g.gfc, g.NGc, g.ncolc, g.NCX,
                       wsc + (size_t)warp * kPch * g.NCX, wcar + (size_t)warp * kPch * (g.NGb + 1), uc, false, mc);
          if (warp == 2) TSTAMP(5);
          int32_t* nxt = CROW(CR_CUR + (par ^ 1) * p.D + m);
          if (warp_normalize_small(uc, g.ncolc, 2, p.W, nxt, &cinfo[CR_CUR + (par ^ 1) * p.D + m], 0) && lane == 0)
            flag[0] = 1;
          if (warp == 2) TSTAMP(6);
          // publish: rows for the bulk warps (after the barrier), state sums
          const bool keep = has_row(m, i + 1);
          int32_t* dst = keep ? ROW(m, i + 1) : nullptr;
          for (int d = lane; d < p.W; d += 32) {
            const int32_t v = nxt[d];
            ssum[(size_t)m * (p.W + 3) + d] += v;
            if (keep) dst[d] = v;
          }
          if (keep && lane == 0) rinfo[SLOT(m, i + 1)] = cinfo[CR_CUR + (par ^ 1) * p.D + m];
          if (p.write_coef && rank == 0) {
            int32_t* gd = p.coef + (((size_t)traj * p.D + m) * (p.N + 1) + i + 1) * p.RS;
            for (int d = lane; d < p.W; d += 32) gd[d] = nxt[d];
            if (i == 0)
              for (int d = lane; d < p.W; d += 32)
                p.coef[(((size_t)traj * p.D + m) * (p.N + 1)) * p.RS + d] = CROW(CR_ZERO + m)[d];
          }
        }
      } else {
        // prefetch tau/(i+2) into the other ctab buffer (read by the chain next order)
        const int bt = tid - 32 * kChainWarps;
        if (i + 1 < p.N)
          for (int d = bt; d < p.W; d += 32 * kBulkWarps)
            CROW(CR_CT + (par ^ 1))[d] = __ldg(p.ctab + (size_t)(i + 1) * p.RS + d);
      }
      if (!is_chain && p.NP > 0) {
        // ================= bulk: P_q(i+1) = sum_{k=1}^{i} a_{i+1-k} b_k, k = rank (mod G)
        const int bt = tid - 32 * kChainWarps;
        const int ns = (32 * kBulkWarps) / g.NGb;
        const int slot = bt / g.NGb, grp = bt - slot * g.NGb;
        // k values of this CTA in [1, i]: k = k1 + G * kk
        const int k1 = rank == 0 ? G : rank;
        const int nk = (i >= k1) ? (i - k1) / G + 1 : 0;
        const int nsa = min(ns, nk);
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
            const int k = k1 + kk * G;
#pragma unroll
            for (int q = 0; q < NPT; q++) {
              if (q < p.NP) {
                const int va = p.pj[q], vb = p.pk[q];
                mac_group(acc[q], cnt[q], ROW(va, i + 1 - k), rinfo[SLOT(va, i + 1 - k)], ROW(vb, k),
                          rinfo[SLOT(vb, k)], c0, g.Tb, mc);
              }
            }
          }
#pragma unroll
          for (int q = 0; q < NPT; q++) {
            if (q < p.NP) {
              acc_fold(acc[q], c0, g.Tb);
              const int u = slot * p.NP + q;
              uint32_t* part = bpart + (size_t)u * g.NCX;
#pragma unroll
              for (int r = 0; r < kR; r++) {
                const int c = c0 + r - g.Tb;
                if (c >= 0) part[c] = (uint32_t)acc[q].v[r];
              }
              bpcar[(size_t)u * g.NGb + grp] = acc[q].v[kR];
            }
          }
        }
        if (warp == kChainWarps) TSTAMP(8);
        asm volatile("bar.sync 2, %0;" ::"r"(32 * kBulkWarps));
        if (warp == kChainWarps) TSTAMP(9);
        // reduce the slots and push the totals into every CTA's receive slot [rank]
        const size_t rbase = (size_t)(par ^ 1) * recv_par;
        for (int w = bt; w < p.NP * g.ncolb; w += 32 * kBulkWarps) {
          const int q = w / g.ncolb, c = w - q * g.ncolb;
          const int64_t s = nsa > 0 ? unit_col(bpart, bpcar, q, p.NP, nsa, g.NCX, g.NGb, c, g.Tb, g.gfb, g.NGb) : 0;
          const size_t off = rbase + ((size_t)rank * NPp + q) * g.ncolb + c;
#pragma unroll 4
          for (int r = 0; r < G; r++) s_recv_remote[r][off] = s;
        }
      }
      // one cluster barrier per order: P(i+1) pushed, coefficient i+1 published
      if (warp == 2) TSTAMP(7);
      if (warp == kChainWarps) TSTAMP(10);
      cluster.sync();
      if (warp == 0) TSTAMP(11);
#undef TSTAMP
    }
    // ---- end of step: state = RN_P(sum of rows) --------------------------------
    if (is_chain) {
      for (int m = warp; m < p.D; m += kChainWarps) {
        if (warp_normalize_small(ssum + (size_t)m * (p.W + 3), p.W + 3, 0, p.W, CROW(CR_ZERO + m), &cinfo[CR_ZERO + m],
                           p.P) &&
            lane == 0)
          flag[0] = 1;
        if (rank == 0 && ((n % p.stride == 0) || (n == p.n_steps))) {
          const int slot = (n % p.stride == 0) ? (n / p.stride - p.start_step / p.stride)
                                               : (p.n_steps / p.stride - p.start_step / p.stride + 1);
          int32_t* dst = p.rec + ((size_t)slot * p.n_traj + traj) * p.D * p.RS + (size_t)m * p.RS;
          for (int d = lane; d < p.W; d += 32) dst[d] = CROW(CR_ZERO + m)[d];
        }
      }
    }
    __syncthreads();
  }
  if (rank == 0)
    for (int m = 0; m < p.D; m++)
      for (int d = tid; d < p.W; d += kThreads) gstate[(size_t)m * p.RS + d] = CROW(CR_ZERO + m)[d];
  __syncthreads();
  if (rank == 0 && tid == 0) p.status[traj] = flag[0] ? kOverflow : kOk;
  if (mc) {
    atomicAdd(&p.counters[0], mcount.useful);
    atomicAdd(&p.counters[1], mcount.executed);
  }
  cluster.sync();
}

}  // namespace pipe

size_t pipe_smem_bytes(const Params& p, int G) { return pipe::make_layout(p, G).total; }

bool pipe_supported(const Params& p) {
  // small/medium precision (warp-level normalisation with <= 8 digits per
  // lane), integer bilinear coefficients, at most kChainWarps equations
  const pipe::Geo g = pipe::make_geo(p);
  return p.D <= pipe::kChainWarps && p.all_q_small && g.ncolb <= 256 && g.ncolc <= 256 &&
         g.NGb * pipe::kPch <= 64;
}

cudaError_t launch_pipe_kernel(const Params& p, int G, size_t smem, cudaStream_t stream) {
  const int npt = p.NP <= 1 ? 1 : p.NP <= 2 ? 2 : 4;
  const void* fn = npt == 1 ? (const void*)pipe::taylor_pipe_kernel<1>
                   : npt == 2 ? (const void*)pipe::taylor_pipe_kernel<2>
                              : (const void*)pipe::taylor_pipe_kernel<4>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (G > 8) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.n_traj * G);
  cfg.blockDim = dim3(pipe::kThreads);
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

int pipe_max_cluster(const Params& p, size_t smem, int want) {
  const void* fn = (const void*)pipe::taylor_pipe_kernel<2>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (want > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(want);
  cfg.blockDim = dim3(pipe::kThreads);
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
