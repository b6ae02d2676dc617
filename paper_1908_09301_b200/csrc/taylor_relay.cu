// Relay kernel: one trajectory per thread-block cluster of G = 2..16 CTAs,
// with the order-to-order critical path on a CTA of its own.
//
//   CTA 0 ("lead")   runs only the recurrence's critical path for order i:
//                      A  new-term products a_i b_0, a_0 b_i (+ non-integer
//                         linear products), split over all 16 warps by
//                         (product, column group, operand slice);
//                      then one 4-warp group per equation m, synchronised by
//                      its own named barrier (no CTA-wide barrier):
//                      B  U_m = sum_t q_t (P_t(i) + new terms) + linear + c_m
//                      C  normalise U_m               (group_normalize)
//                      D  U_m (x) tau/(i+1)           (128 threads)
//                      E  normalise -> coefficient i+1, publish it into the
//                         rows of the bulk CTAs (st.shared::cluster), add it
//                         to the state sum
//   CTAs 1..G-1      compute the lookahead part P_q(i+1) = sum_{k=1}^{i}
//   ("bulk")           a_{i+1-k} b_k for k = b (mod G-1), all 16 warps, and
//                      push their column sums into the lead's receive buffer.
//   ---- one cluster barrier per order.
//
// Compared with the pipe kernel (taylor_pipe.cu) the lead's warps no longer
// share issue slots with bulk warps, and every chain step is spread over 4-16
// warps instead of one. Arithmetic is identical to oracle/fixmodel.c (exact
// column sums, same roundings), so the result bits do not change.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "mpt_common.cuh"
#include "mpt_device.cuh"

namespace cg = cooperative_groups;

namespace mpt {
namespace relay {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kGW = 4;  // warps per equation group on the lead CTA
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

__host__ __device__ inline int n_lin_big(const Params& p) {
  int n = 0;
  for (int t = 0; t < p.D * p.D; t++) n += p.lin_small[t] ? 0 : 1;
  return n;
}

struct Layout {
  int rs, Gb, nprod, pcha, pchc, ns;
  // lead CTA
  size_t off_crow, off_cinfo, off_recv, off_apart, off_apcar, off_cpart, off_cpcar, off_ucol, off_ssum, off_xs,
      off_flag, lead_total;
  // bulk CTAs
  int nslots, base[kMaxD], full[kMaxD];
  size_t off_rows, off_rinfo, off_bpart, off_bpcar, bulk_total;
  size_t total;
};

// lead crow rows: CST D | LIN D*D | CT 2 | ZERO D | CUR 2D | U D
__host__ __device__ inline Layout make_layout(const Params& p, int G) {
  Layout L;
  const Geo g = make_geo(p);
  const int NPp = p.NP > 0 ? p.NP : 1;
  L.rs = (p.W + 3) / 4 * 4 + kPad + 1;
  L.Gb = G - 1;
  L.nprod = 2 * p.NP + n_lin_big(p);
  const int np1 = L.nprod > 0 ? L.nprod : 1;
  L.pcha = kThreads / (np1 * g.NGb);
  L.pcha = L.pcha < 1 ? 1 : (L.pcha > 16 ? 16 : L.pcha);
  L.pchc = (32 * kGW) / g.NGc;
  L.pchc = L.pchc < 1 ? 1 : (L.pchc > 16 ? 16 : L.pchc);
  L.ns = kThreads / g.NGb;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o += (bytes + 15) / 16 * 16;
    return r;
  };
  const int ncrow = p.D + p.D * p.D + 2 + p.D + 2 * p.D + p.D;
  L.off_crow = take(sizeof(int32_t) * ((size_t)ncrow * L.rs + kPad));
  L.off_cinfo = take(sizeof(int2) * (size_t)ncrow);
  L.off_recv = take(sizeof(int64_t) * 2 * (size_t)(L.Gb > 0 ? L.Gb : 1) * NPp * g.ncolb);
  L.off_apart = take(sizeof(uint32_t) * (size_t)np1 * L.pcha * g.NCX);
  L.off_apcar = take(sizeof(int64_t) * (size_t)np1 * L.pcha * g.NGb);
  L.off_cpart = take(sizeof(uint32_t) * (size_t)kMaxD * L.pchc * g.NCX);
  L.off_cpcar = take(sizeof(int64_t) * (size_t)kMaxD * L.pchc * g.NGc);
  L.off_ucol = take(sizeof(int64_t) * (size_t)kMaxD * g.NCX);
  L.off_ssum = take(sizeof(int64_t) * (size_t)p.D * (p.W + 3));
  L.off_xs = take(sizeof(int64_t) * kMaxD * 32);
  L.off_flag = take(sizeof(int) * 8);
  L.lead_total = o;
  // bulk: rows of left-hand pair variables for every order, right-hand rows
  // only for k = b (mod Gb)
  o = 0;
  int s = 0;
  for (int v = 0; v < p.D; v++) {
    int is_left = 0;
    for (int q = 0; q < p.NP; q++) is_left |= (p.pj[q] == v);
    L.full[v] = is_left || L.Gb <= 1;
    L.base[v] = s;
    s += L.full[v] ? p.N + 1 : (p.N + L.Gb) / L.Gb + 1;
  }
  L.nslots = s;
  L.off_rows = take(sizeof(int32_t) * ((size_t)L.nslots * L.rs + 2 * kPad));
  L.off_rinfo = take(sizeof(int2) * (size_t)L.nslots);
  L.off_bpart = take(sizeof(uint32_t) * (size_t)L.ns * NPp * g.NCX);
  L.off_bpcar = take(sizeof(int64_t) * (size_t)L.ns * NPp * g.NGb);
  L.bulk_total = o;
  L.total = L.lead_total > L.bulk_total ? L.lead_total : L.bulk_total;
  return L;
}

__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int NPT>
__global__ void __launch_bounds__(kThreads, 1) taylor_relay_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(16) unsigned char smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int G = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int traj = blockIdx.x / G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Geo g = make_geo(p);
  const Layout L = make_layout(p, G);
  const int NPp = p.NP > 0 ? p.NP : 1;
  const int Gb = L.Gb;
  const int rs = L.rs;
  MacCount mcount;
  MacCount* mc = p.counters ? &mcount : nullptr;

  for (size_t w = tid; w < L.total / 4; w += kThreads) ((int32_t*)smem)[w] = 0;
  __shared__ int s_base[kMaxD], s_full[kMaxD];
  if (tid < kMaxD) {
    s_base[tid] = tid < p.D ? L.base[tid] : 0;
    s_full[tid] = tid < p.D ? L.full[tid] : 1;
  }
  // bulk-layout row addressing (valid in every CTA; rows live in bulk CTAs)
  auto SLOT = [&](int v, int k) { return s_base[v] + (s_full[v] ? k : k / Gb); };
  int32_t* rows = (int32_t*)(smem + L.off_rows) + kPad;
  int2* rinfo = (int2*)(smem + L.off_rinfo);

  if (rank == 0) {
    // =============================== lead CTA ===============================
    int32_t* crow = (int32_t*)(smem + L.off_crow) + kPad;
    int2* cinfo = (int2*)(smem + L.off_cinfo);
    int64_t* recv = (int64_t*)(smem + L.off_recv);
    uint32_t* apart = (uint32_t*)(smem + L.off_apart);
    int64_t* apcar = (int64_t*)(smem + L.off_apcar);
    uint32_t* cpart = (uint32_t*)(smem + L.off_cpart);
    int64_t* cpcar = (int64_t*)(smem + L.off_cpcar);
    int64_t* ucol = (int64_t*)(smem + L.off_ucol);
    int64_t* ssum = (int64_t*)(smem + L.off_ssum);
    int64_t* xs = (int64_t*)(smem + L.off_xs);
    int* flag = (int*)(smem + L.off_flag);
    const int CR_CST = 0, CR_LIN = p.D, CR_CT = CR_LIN + p.D * p.D, CR_ZERO = CR_CT + 2, CR_CUR = CR_ZERO + p.D,
              CR_U = CR_CUR + 2 * p.D;
    auto CROW = [&](int r) { return crow + (size_t)r * rs; };
    __shared__ int s_lin_it[kMaxD * kMaxD];
    __shared__ int32_t* s_rows_remote[kMaxG];
    __shared__ int2* s_rinfo_remote[kMaxG];
    if (tid < kMaxG) {
      s_rows_remote[tid] = (tid >= 1 && tid < G) ? cluster.map_shared_rank(rows, tid) : nullptr;
      s_rinfo_remote[tid] = (tid >= 1 && tid < G) ? cluster.map_shared_rank(rinfo, tid) : nullptr;
    }
    if (tid == 0) {
      int n = 0;
      for (int t = 0; t < p.D * p.D; t++)
        if (!p.lin_small[t]) s_lin_it[n++] = t;
    }
    __syncthreads();
    for (int r = 0; r < CR_CT; r++) {
      const int32_t* src = r < CR_LIN ? p.cst + (size_t)r * p.RS : p.lin + (size_t)(r - CR_LIN) * p.RS;
      for (int d = tid; d < p.W; d += kThreads) CROW(r)[d] = src[d];
    }
    int32_t* gstate = p.state + (size_t)traj * p.D * p.RS;
    for (int m = 0; m < p.D; m++)
      for (int d = tid; d < p.W; d += kThreads) CROW(CR_ZERO + m)[d] = gstate[(size_t)m * p.RS + d];
    __syncthreads();
    for (int r = warp; r < CR_CT; r += kWarps) {
      int2 inf = make_int2(1 << 30, -1);
      for (int d = lane; d < p.W; d += 32)
        if (CROW(r)[d]) {
          inf.x = min(inf.x, d);
          inf.y = max(inf.y, d);
        }
      inf.x = __reduce_min_sync(0xffffffffu, inf.x);
      inf.y = __reduce_max_sync(0xffffffffu, inf.y);
      if (lane == 0) cinfo[r] = make_int2(inf.y >= 0 ? inf.x : p.W, inf.y);
    }
    const int nlb = L.nprod - 2 * p.NP;
    const int geq = warp / kGW, gw = warp % kGW, gt = gw * 32 + lane;
    const int bar_id = 1 + geq;
    cluster.sync();

    for (int n = p.start_step + 1; n <= p.n_steps; n++) {
      // ---- order 0: CUR parity 0 = ZERO = state; state sum restarts; C_0
      for (int m = 0; m < p.D; m++)
        for (int d = tid; d < p.W + 3; d += kThreads) {
          const int32_t v = d < p.W ? CROW(CR_ZERO + m)[d] : 0;
          ssum[(size_t)m * (p.W + 3) + d] = v;
          if (d < p.W) CROW(CR_CUR + m)[d] = v;
        }
      for (int d = tid; d < p.W; d += kThreads) CROW(CR_CT)[d] = __ldg(p.ctab + d);
      __syncthreads();
      if (warp < p.D) {
        int2 inf = make_int2(1 << 30, -1);
        for (int d = lane; d < p.W; d += 32)
          if (CROW(CR_ZERO + warp)[d]) {
            inf.x = min(inf.x, d);
            inf.y = max(inf.y, d);
          }
        inf.x = __reduce_min_sync(0xffffffffu, inf.x);
        inf.y = __reduce_max_sync(0xffffffffu, inf.y);
        if (lane == 0) {
          const int2 v = make_int2(inf.y >= 0 ? inf.x : p.W, inf.y);
          cinfo[CR_ZERO + warp] = v;
          cinfo[CR_CUR + warp] = v;
        }
      }
      __syncthreads();

      for (int i = 0; i < p.N; i++) {
        const int par = i & 1;
        const bool tlog = p.dbg && n == p.start_step + 1 && i < 200 && lane == 0;
#define TSTAMP(ev) \
  if (tlog) p.dbg[(size_t)i * 16 + (ev)] = (long long)clock64();
        if (warp == 0) TSTAMP(0);
        const int32_t* cur = CROW(CR_CUR + par * p.D);
        const int2* curinf = cinfo + CR_CUR + par * p.D;
        // ---- A: new-term products over all warps; info of this order's C_i row
        if (warp == kWarps - 1) {
          int2 inf = make_int2(1 << 30, -1);
          for (int d = lane; d < p.W; d += 32)
            if (CROW(CR_CT + par)[d]) {
              inf.x = min(inf.x, d);
              inf.y = max(inf.y, d);
            }
          inf.x = __reduce_min_sync(0xffffffffu, inf.x);
          inf.y = __reduce_max_sync(0xffffffffu, inf.y);
          if (lane == 0) cinfo[CR_CT + par] = make_int2(inf.y >= 0 ? inf.x : p.W, inf.y);
        }
        {
          const int per_prod = g.NGb * L.pcha;
          for (int e = tid; e < L.nprod * per_prod; e += kThreads) {
            const int pr = e / per_prod, rem = e - pr * per_prod, grp = rem / L.pcha, pc = rem - grp * L.pcha;
            const int c0 = kR * (g.gfb + grp);
            Acc acc;
            acc_zero(acc);
            const int32_t *A = nullptr, *B = nullptr;
            int2 ia = make_int2(0, -1), ib = make_int2(0, -1);
            if (pr < 2 * p.NP) {
              const int q = pr >> 1, va = p.pj[q], vb = p.pk[q];
              if ((pr & 1) == 0) {  // a_i b_0
                A = cur + (size_t)va * rs;
                ia = curinf[va];
                B = CROW(CR_ZERO + vb);
                ib = cinfo[CR_ZERO + vb];
              } else if (i > 0) {  // a_0 b_i
                A = CROW(CR_ZERO + va);
                ia = cinfo[CR_ZERO + va];
                B = cur + (size_t)vb * rs;
                ib = curinf[vb];
              }
            } else {
              const int it = s_lin_it[pr - 2 * p.NP], j = it % p.D;
              A = CROW(CR_LIN + it);
              ia = cinfo[CR_LIN + it];
              B = cur + (size_t)j * rs;
              ib = curinf[j];
            }
            if (A != nullptr && ia.y >= 0 && ib.y >= 0) {
              int cnt = 0;
              mac_group_chunk(acc, cnt, A, ia, B, ib, c0, g.Tb, pc, L.pcha, mc);
              acc_fold(acc, c0, g.Tb);
            }
            const int u = pr * L.pcha + pc;
            unit_store(apart + (size_t)u * g.NCX, apcar + (size_t)u * g.NGb, acc, grp, c0, g.Tb);
          }
        }
        __syncthreads();
        if (warp == 0) TSTAMP(1);
        if (geq < p.D) {
          const int m = geq;
          int64_t* uc = ucol + (size_t)m * g.NCX;
          // ---- B: numerator columns
          const int64_t* rv = recv + (size_t)par * Gb * NPp * g.ncolb;
          for (int c = gt; c < g.ncolb; c += 32 * kGW) {
            int64_t s = 0;
            for (int t = 0; t < p.NT; t++) {
              if (p.teq[t] != m) continue;
              const int q = p.tpair[t];
              int64_t v = unit_column(apart, apcar, 2 * q * L.pcha, 1, 2 * L.pcha, g.NCX, g.NGb, c, g.Tb, g.gfb,
                                      g.NGb);
              if (i >= 2) {
#pragma unroll 4
                for (int r = 0; r < Gb; r++) v += rv[((size_t)r * NPp + q) * g.ncolb + c];
              }
              s += (int64_t)p.tq_int[t] * v;
            }
            for (int l = 0; l < nlb; l++)
              if (s_lin_it[l] / p.D == m)
                s += unit_column(apart, apcar, (2 * p.NP + l) * L.pcha, 1, L.pcha, g.NCX, g.NGb, c, g.Tb, g.gfb,
                                 g.NGb);
            if (c >= 2 && c - 2 < p.W) {
              const int dgt = c - 2;
              if (i == 0) s += CROW(CR_CST + m)[dgt];
              for (int j = 0; j < p.D; j++)
                if (p.lin_small[m * p.D + j]) s += (int64_t)p.lin_int[m * p.D + j] * cur[(size_t)j * rs + dgt];
            }
            uc[c] = s;
          }
          group_sync(bar_id, 32 * kGW);
          if (gt == 0 && m == 0) TSTAMP(2);
          // ---- C: U_m = rnd(numerator)
          if (group_normalize(uc, g.ncolb, 2, p.W, CROW(CR_U + m), &cinfo[CR_U + m], 0, gw, kGW, bar_id,
                              xs + 32 * m) &&
              gt == 0)
            flag[0] = 1;
          if (gt == 0 && m == 0) TSTAMP(3);
          // ---- D: U_m (x) tau/(i+1)
          {
            const int32_t* U = CROW(CR_U + m);
            const int2 uinf = cinfo[CR_U + m];
            const int32_t* ct = CROW(CR_CT + par);
            const int2 ctinf = cinfo[CR_CT + par];
            uint32_t* cp = cpart + (size_t)m * L.pchc * g.NCX;
            int64_t* cc = cpcar + (size_t)m * L.pchc * g.NGc;
            for (int e = gt; e < g.NGc * L.pchc; e += 32 * kGW) {
              const int grp = e / L.pchc, pc = e - grp * L.pchc;
              const int c0 = kR * (g.gfc + grp);
              Acc acc;
              acc_zero(acc);
              if (uinf.y >= 0 && ctinf.y >= 0) {
                int cnt = 0;
                mac_group_chunk(acc, cnt, U, uinf, ct, ctinf, c0, g.Tc, pc, L.pchc, mc);
                acc_fold(acc, c0, g.Tc);
              }
              unit_store(cp + (size_t)pc * g.NCX, cc + (size_t)pc * g.NGc, acc, grp, c0, g.Tc);
            }
            group_sync(bar_id, 32 * kGW);
            for (int c = gt; c < g.ncolc; c += 32 * kGW)
              uc[c] = unit_column(cp, cc, 0, 1, L.pchc, g.NCX, g.NGc, c, g.Tc, g.gfc, g.NGc);
            group_sync(bar_id, 32 * kGW);
          }
          if (gt == 0 && m == 0) TSTAMP(4);
          // ---- E: coefficient i+1 of variable m
          int32_t* nxt = CROW(CR_CUR + (par ^ 1) * p.D + m);
          int2* nxtinf = &cinfo[CR_CUR + (par ^ 1) * p.D + m];
          if (group_normalize(uc, g.ncolc, 2, p.W, nxt, nxtinf, 0, gw, kGW, bar_id, xs + 32 * m) && gt == 0)
            flag[0] = 1;
          if (gt == 0 && m == 0) TSTAMP(5);
          const int k = i + 1;
          const int slot = SLOT(m, k);
          const int b_only = s_full[m] ? -1 : 1 + (k % Gb);
          for (int d = gt; d < p.W; d += 32 * kGW) {
            const int32_t v = nxt[d];
            ssum[(size_t)m * (p.W + 3) + d] += v;
            if (b_only > 0) {
              s_rows_remote[b_only][(size_t)slot * rs + d] = v;
            } else {
              for (int r = 1; r < G; r++) s_rows_remote[r][(size_t)slot * rs + d] = v;
            }
          }
          if (gt < G && gt >= 1 && (b_only < 0 || gt == b_only)) s_rinfo_remote[gt][slot] = *nxtinf;
          if (p.write_coef) {
            int32_t* gd = p.coef + (((size_t)traj * p.D + m) * (p.N + 1) + k) * p.RS;
            for (int d = gt; d < p.W; d += 32 * kGW) gd[d] = nxt[d];
            if (i == 0)
              for (int d = gt; d < p.W; d += 32 * kGW)
                p.coef[(((size_t)traj * p.D + m) * (p.N + 1)) * p.RS + d] = CROW(CR_ZERO + m)[d];
          }
          if (gt == 0 && m == 0) TSTAMP(6);
        }
        // prefetch tau/(i+2) into the other C buffer (read after the barrier)
        if (i + 1 < p.N)
          for (int d = tid; d < p.W; d += kThreads) CROW(CR_CT + (par ^ 1))[d] = __ldg(p.ctab + (size_t)(i + 1) * p.RS + d);
        cluster_arrive_release();
        cluster_wait_acquire();
        if (warp == 0) TSTAMP(7);
#undef TSTAMP
      }
      // ---- end of step: state = RN_P(sum of rows)
      __syncthreads();
      if (geq < p.D) {
        const int m = geq;
        if (group_normalize(ssum + (size_t)m * (p.W + 3), p.W + 3, 0, p.W, CROW(CR_ZERO + m), &cinfo[CR_ZERO + m],
                            p.P, gw, kGW, bar_id, xs + 32 * m) &&
            gt == 0)
          flag[0] = 1;
        if ((n % p.stride == 0) || (n == p.n_steps)) {
          const int slot = (n % p.stride == 0) ? (n / p.stride - p.start_step / p.stride)
                                               : (p.n_steps / p.stride - p.start_step / p.stride + 1);
          int32_t* dst = p.rec + ((size_t)slot * p.n_traj + traj) * p.D * p.RS + (size_t)m * p.RS;
          for (int d = gt; d < p.W; d += 32 * kGW) dst[d] = CROW(CR_ZERO + m)[d];
        }
      }
      __syncthreads();
    }
    for (int m = 0; m < p.D; m++)
      for (int d = tid; d < p.W; d += kThreads) gstate[(size_t)m * p.RS + d] = CROW(CR_ZERO + m)[d];
    __syncthreads();
    if (tid == 0) p.status[traj] = flag[0] ? kOverflow : kOk;
  } else {
    // =============================== bulk CTA ===============================
    const int b = rank - 1;
    uint32_t* bpart = (uint32_t*)(smem + L.off_bpart);
    int64_t* bpcar = (int64_t*)(smem + L.off_bpcar);
    int64_t* lead_recv = cluster.map_shared_rank((int64_t*)(smem + L.off_recv), 0);
    __syncthreads();
    cluster.sync();
    const int k1 = b == 0 ? Gb : b;  // smallest k >= 1 with k = b (mod Gb)
    const int slot0 = tid / g.NGb, grp = tid - slot0 * g.NGb;
    for (int n = p.start_step + 1; n <= p.n_steps; n++) {
      for (int i = 0; i < p.N; i++) {
        const int par = i & 1;
        const bool tlog = p.dbg && n == p.start_step + 1 && i < 200 && lane == 0 && rank == 1;
        const int nk = (i >= k1) ? (i - k1) / Gb + 1 : 0;
        if (nk > 0 && p.NP > 0) {
          int pch = L.ns / nk;
          pch = pch < 1 ? 1 : (pch > 8 ? 8 : pch);
          const int nks = L.ns / pch;  // k slots
          const int nsa = (nks < nk ? nks : nk) * pch;
          if (slot0 < nsa) {
            const int ks = slot0 / pch, pc = slot0 - ks * pch;
            const int c0 = kR * (g.gfb + grp);
            Acc acc[NPT];
            int cnt[NPT];
#pragma unroll
            for (int q = 0; q < NPT; q++) {
              acc_zero(acc[q]);
              cnt[q] = 0;
            }
            for (int kk = ks; kk < nk; kk += nks) {
              const int k = k1 + kk * Gb;
#pragma unroll
              for (int q = 0; q < NPT; q++) {
                if (q < p.NP) {
                  const int va = p.pj[q], vb = p.pk[q];
                  const int sa = SLOT(va, i + 1 - k), sb = SLOT(vb, k);
                  mac_group_chunk(acc[q], cnt[q], rows + (size_t)sa * rs, rinfo[sa], rows + (size_t)sb * rs,
                                  rinfo[sb], c0, g.Tb, pc, pch, mc);
                }
              }
            }
#pragma unroll
            for (int q = 0; q < NPT; q++) {
              if (q < p.NP) {
                acc_fold(acc[q], c0, g.Tb);
                const int u = slot0 * p.NP + q;
                unit_store(bpart + (size_t)u * g.NCX, bpcar + (size_t)u * g.NGb, acc[q], grp, c0, g.Tb);
              }
            }
          }
          if (tlog && warp == 0) p.dbg[(size_t)i * 16 + 8] = (long long)clock64();
          __syncthreads();
          // column sums of P_q(i+1) -> lead's receive slot [b], parity (i+1)&1
          int64_t* dst = lead_recv + (size_t)(par ^ 1) * Gb * NPp * g.ncolb + (size_t)b * NPp * g.ncolb;
          for (int w = tid; w < p.NP * g.ncolb; w += kThreads) {
            const int q = w / g.ncolb, c = w - q * g.ncolb;
            dst[(size_t)q * g.ncolb + c] =
                unit_column(bpart, bpcar, q, p.NP, nsa, g.NCX, g.NGb, c, g.Tb, g.gfb, g.NGb);
          }
        } else if (i >= 1 && p.NP > 0) {
          // no k of this CTA in [1, i]: its share of P(i+1) is zero
          int64_t* dst = lead_recv + (size_t)(par ^ 1) * Gb * NPp * g.ncolb + (size_t)b * NPp * g.ncolb;
          for (int w = tid; w < p.NP * g.ncolb; w += kThreads) dst[w] = 0;
        }
        if (tlog && warp == 0) p.dbg[(size_t)i * 16 + 9] = (long long)clock64();
        cluster_arrive_release();
        cluster_wait_acquire();
        __syncthreads();  // bpart reuse next order
      }
    }
  }
  if (mc) {
    atomicAdd(&p.counters[0], mcount.useful);
    atomicAdd(&p.counters[1], mcount.executed);
  }
  cluster.sync();
}

}  // namespace relay

size_t relay_smem_bytes(const Params& p, int G) { return relay::make_layout(p, G).total; }

bool relay_supported(const Params& p) {
  const relay::Geo g = relay::make_geo(p);
  return p.D <= kMaxD && p.all_q_small && p.NP <= 4 && g.ncolb <= 2048 && g.ncolc <= 2048;
}

cudaError_t launch_relay_kernel(const Params& p, int G, size_t smem, cudaStream_t stream) {
  const int npt = p.NP <= 1 ? 1 : p.NP <= 2 ? 2 : 4;
  const void* fn = npt == 1 ? (const void*)relay::taylor_relay_kernel<1>
                   : npt == 2 ? (const void*)relay::taylor_relay_kernel<2>
                              : (const void*)relay::taylor_relay_kernel<4>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (G > 8) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.n_traj * G);
  cfg.blockDim = dim3(relay::kThreads);
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

int relay_max_cluster(const Params& p, size_t smem, int want) {
  const void* fn = (const void*)relay::taylor_relay_kernel<2>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (want > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(want);
  cfg.blockDim = dim3(relay::kThreads);
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
