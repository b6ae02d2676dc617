// C ABI of the B200 Taylor engine: plan construction, constant upload,
// launches. See include/mptaylor_b200.h for the contract.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mptaylor_b200.h"
#include "mpt_common.cuh"

namespace mpt {
size_t smem_bytes(const Params& p);
cudaError_t launch_team_kernel(const Params& p, size_t smem, cudaStream_t stream);
cudaError_t launch_imad_probe(int blocks, int threads, int iters, long long* out, cudaStream_t s);
bool grid_supported(const Params& p);
size_t grid_smem_bytes(const Params& p, int kc);
size_t grid_scratch_bytes(const Params& p);
cudaError_t launch_grid_kernel(const Params& p, int nblocks, int kc, size_t smem, cudaStream_t stream);
int grid_max_blocks(const Params& p, size_t smem);
size_t mx_smem_bytes(const Params& p, int G);
size_t mx_scratch_bytes(const Params& p);
bool mx_supported(const Params& p);
cudaError_t launch_mx_kernel(const Params& p, int G, size_t smem, cudaStream_t stream);
int mx_max_cluster(const Params& p, size_t smem, int want);
bool warp_supported(const Params& p);
size_t warp_traj_smem(const Params& p);
int warp_choose_wpb(const Params& p, size_t smem_sm, size_t optin);
cudaError_t launch_warp_kernel(const Params& p, int wpb, cudaStream_t stream);
bool block_supported(const Params& p);
size_t block_smem_bytes(const Params& p);
cudaError_t launch_block_kernel(const Params& p, cudaStream_t stream);
bool cblock_supported(const Params& p);
size_t cblock_smem_bytes(const Params& p, int G);
int cblock_max_clusters(const Params& p, size_t smem, int G);
cudaError_t launch_cblock_kernel(const Params& p, int G, size_t smem, cudaStream_t stream);
}  // namespace mpt

static thread_local std::string g_err;
static long long* g_dbg = nullptr;  // MPT_DEBUG dump buffer (development only)

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(MPT_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));        \
  } while (0)

struct mpt_plan {
  mpt::Params p;
  int device = 0;
  int W = 0;
  size_t smem = 0;
  int32_t *d_cst = nullptr, *d_lin = nullptr, *d_q = nullptr, *d_ctab = nullptr;
  int32_t *d_coef = nullptr, *d_state = nullptr, *d_rec = nullptr, *d_status = nullptr;
  int2* d_rinfo = nullptr;
  size_t rec_slots = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  float last_ms = 0.f;
  bool have_constants = false;
  unsigned long long* d_counters = nullptr;
  bool counting = false;
  int kernel = 0;    // 1 team (rows in HBM/L2), 4 grid (all SMs), 6 mx (matrix recurrence), 7 warp (one warp per trajectory),
                     // 8 block (one CTA per trajectory, rows in shared memory), 9 cblock (one cluster per trajectory,
                     // rows in every CTA's shared memory, all-gather of partial Cauchy sums)
  int warp_wpb = 0;  // warp kernel: trajectories (warps) per CTA
  int smem_sm = 0;   // shared memory per SM
  int cluster = 1;   // CTAs per trajectory (mx), co-resident CTAs (grid)
  size_t smem_cluster = 0;
  int optin = 0;
  int nsm = 148;     // SMs of the device
  int requested_kernel = 0, requested_cluster = 1;
  int grid_blocks = 0, grid_kc = 0;
  size_t smem_grid = 0;
  void* d_gscratch = nullptr;
  void* d_mxscratch = nullptr;
  size_t mxscratch_bytes = 0;
};

static int setup_grid(mpt_plan* pl) {
  mpt::Params& p = pl->p;
  int kc = 64;
  size_t s = 0;
  for (; kc >= 1; kc = kc > 8 ? kc - 8 : kc - 1) {
    s = mpt::grid_smem_bytes(p, kc);
    if (s <= (size_t)pl->optin) break;
  }
  if (kc < 1) return fail(MPT_EUNSUP, "grid kernel: shared memory budget exceeded");
  int nb = mpt::grid_max_blocks(p, s);
  if (nb < 1) return fail(MPT_EUNSUP, "grid kernel: no co-resident blocks");
  if (!pl->d_gscratch) {
    CK(cudaMalloc(&pl->d_gscratch, mpt::grid_scratch_bytes(p)));
    CK(cudaMemset(pl->d_gscratch, 0, mpt::grid_scratch_bytes(p)));
  }
  p.gscratch = pl->d_gscratch;
  pl->grid_blocks = nb;
  pl->grid_kc = kc;
  pl->smem_grid = s;
  return MPT_OK;
}

// choose the kernel (0 = automatic): one trajectory -> mx (cluster of `want` CTAs,
// clamped to what co-schedules) when the system fits it, else the grid kernel on
// every SM; ensembles -> team (one CTA per trajectory)
static int choose_kernel(mpt_plan* pl, int kernel, int want) {
  mpt::Params& p = pl->p;
  pl->requested_kernel = kernel;
  pl->requested_cluster = want;
  if (kernel == 1) {
    pl->kernel = 1;
    pl->cluster = 1;
    return MPT_OK;
  }
  if (kernel == 4) {
    if (!pl->have_constants) {
      pl->kernel = 0;
      return MPT_OK;
    }
    if (!mpt::grid_supported(p)) return fail(MPT_EUNSUP, "grid kernel: one trajectory, integer bilinear coefficients");
    int rc = setup_grid(pl);
    if (rc) return rc;
    pl->kernel = 4;
    pl->cluster = pl->grid_blocks;
    return MPT_OK;
  }
  // small precision (W <= 34 digits): one warp per trajectory, rows in shared memory
  if ((kernel == 0 || kernel == 7) && pl->have_constants && mpt::warp_supported(p)) {
    const int wpb = mpt::warp_choose_wpb(p, (size_t)pl->smem_sm, (size_t)pl->optin);
    if (wpb > 0) {
      pl->kernel = 7;
      pl->cluster = 1;
      pl->warp_wpb = p.n_traj < wpb ? p.n_traj : wpb;
      pl->smem_cluster = mpt::warp_traj_smem(p) * pl->warp_wpb;
      return MPT_OK;
    }
  }
  if (kernel == 7) {
    if (!pl->have_constants) {
      pl->kernel = 0;
      return MPT_OK;
    }
    return fail(MPT_EUNSUP, "the warp kernel does not support this system/precision (W <= 34 digits, integer bilinear coefficients, rows in shared memory)");
  }
  // medium precision ensembles (35..58 digits): one CTA per trajectory, rows in shared memory
  if ((kernel == 8 || (kernel == 0 && p.n_traj >= pl->nsm / 2)) && pl->have_constants && mpt::block_supported(p) &&
      mpt::block_smem_bytes(p) <= (size_t)pl->optin) {
    pl->kernel = 8;
    pl->cluster = 1;
    pl->smem_cluster = mpt::block_smem_bytes(p);
    return MPT_OK;
  }
  if (kernel == 8) {
    if (!pl->have_constants) {
      pl->kernel = 0;
      return MPT_OK;
    }
    return fail(MPT_EUNSUP, "the block kernel does not support this system/precision (W <= 58 digits, <= 2 integer-coefficient pairs, rows in shared memory)");
  }
  const int tries[] = {16, 8, 4, 2, 1};
  // medium precision, few trajectories: one cluster per trajectory, rows in every CTA's shared memory
  if (kernel == 9 && pl->have_constants &&
      mpt::cblock_supported(p)) {
    for (int G : tries) {
      if (G > want) continue;
      const size_t s = mpt::cblock_smem_bytes(p, G);
      if (s > (size_t)pl->optin) continue;
      if (mpt::cblock_max_clusters(p, s, G) < 1) continue;
      pl->kernel = 9;
      pl->cluster = G;
      pl->smem_cluster = s;
      return MPT_OK;
    }
  }
  if (kernel == 9) {
    if (!pl->have_constants) {
      pl->kernel = 0;
      return MPT_OK;
    }
    return fail(MPT_EUNSUP, "the cblock kernel does not support this system/precision (W <= 93 digits, <= 2 integer-coefficient pairs, rows in shared memory)");
  }
  // the matrix-recurrence kernel (lead CTA + bulk CTAs, K table in global memory)
  if ((kernel == 0 || kernel == 6) && pl->have_constants && mpt::mx_supported(p) && (kernel == 6 || p.n_traj == 1)) {
    for (int G : tries) {
      if (G > want || G < 2) continue;
      size_t s = mpt::mx_smem_bytes(p, G);
      if (s > (size_t)pl->optin) continue;
      if (mpt::mx_max_cluster(p, s, G) < 1) continue;
      const size_t need = mpt::mx_scratch_bytes(p);
      if (need > pl->mxscratch_bytes) {
        cudaFree(pl->d_mxscratch);
        pl->d_mxscratch = nullptr;
        pl->mxscratch_bytes = 0;
        CK(cudaMalloc(&pl->d_mxscratch, need));
        pl->mxscratch_bytes = need;
      }
      pl->kernel = 6;
      pl->cluster = G;
      pl->smem_cluster = s;
      return MPT_OK;
    }
  }
  if (kernel == 6) {
    if (!pl->have_constants) {
      pl->kernel = 0;
      return MPT_OK;
    }
    return fail(MPT_EUNSUP, "the mx kernel does not support this system/precision");
  }
  // ensembles that fill every SM: one trajectory per CTA (team kernel, two
  // CTAs per SM) beats a per-trajectory cluster (measured ens100-ens800)
  if (kernel == 0 && p.n_traj >= pl->nsm) {
    pl->kernel = 1;
    pl->cluster = 1;
    return MPT_OK;
  }
  if (kernel == 0 && pl->have_constants && mpt::grid_supported(p) && setup_grid(pl) == MPT_OK) {
    pl->kernel = 4;
    pl->cluster = pl->grid_blocks;
    return MPT_OK;
  }
  pl->kernel = 1;
  pl->cluster = 1;
  return MPT_OK;
}

extern "C" {

int mpt_version(void) { return 1; }
const char* mpt_last_error(void) { return g_err.c_str(); }

int mpt_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int mpt_record_count(int n_steps, int start_step, int stride) {
  if (stride < 1 || n_steps < start_step) return MPT_EINVAL;
  // records: start_step, every multiple of stride in (start_step, n_steps], and
  // n_steps itself when it is not one of them (taylor.py:202 integrate)
  int n = 1 + (n_steps / stride - start_step / stride);
  if (n_steps % stride && n_steps > start_step) n += 1;
  return n;
}

int mpt_plan_create(mpt_plan** out, int dim, int nterms, const int32_t* term_eq, const int32_t* term_j,
                    const int32_t* term_k, int frac_digits, int c_shift, int order, int prec_bits,
                    int n_traj, int device) {
  if (!out) return fail(MPT_EINVAL, "null plan pointer");
  *out = nullptr;
  if (mpt_device_count() <= 0) return fail(MPT_ENODEV, "no CUDA device available");
  if (dim < 1 || dim > mpt::kMaxD) return fail(MPT_EUNSUP, "dim must be in [1, 4] on the device");
  if (nterms < 0 || nterms > mpt::kMaxT) return fail(MPT_EUNSUP, "too many bilinear terms");
  if (frac_digits < 3 || order < 1 || n_traj < 1 || (c_shift != 0 && c_shift != 1) || prec_bits < 1)
    return fail(MPT_EINVAL, "invalid plan dimensions");
  if (frac_digits + 4 > 32 * mpt::kMaxLanesDigits - 8)
    return fail(MPT_EUNSUP, "precision too large for the device normaliser");
  mpt_plan* pl = new mpt_plan();
  mpt::Params& p = pl->p;
  std::memset(&p, 0, sizeof(p));
  p.D = dim;
  p.NT = nterms;
  p.Lf = frac_digits;
  p.W = frac_digits + 1;
  p.RS = (p.W + 3) / 4 * 4;
  p.sc = c_shift;
  p.N = order;
  p.P = prec_bits;
  p.n_traj = n_traj;
  p.nthreads = 256;
  // distinct pairs in first-appearance order (systems.py:65 product_pairs)
  for (int t = 0; t < nterms; t++) {
    if (term_eq[t] < 0 || term_eq[t] >= dim || term_j[t] < 0 || term_k[t] < term_j[t] || term_k[t] >= dim) {
      delete pl;
      return fail(MPT_EINVAL, "bad bilinear term indices");
    }
    int q = -1;
    for (int r = 0; r < p.NP; r++)
      if (p.pj[r] == term_j[t] && p.pk[r] == term_k[t]) q = r;
    if (q < 0) {
      if (p.NP >= mpt::kMaxP) {
        delete pl;
        return fail(MPT_EUNSUP, "too many distinct product pairs");
      }
      q = p.NP++;
      p.pj[q] = term_j[t];
      p.pk[q] = term_k[t];
    }
    p.teq[t] = term_eq[t];
    p.tpair[t] = q;
  }
  for (int q = 0; q < p.NP; q++) {
    int a = -1, b = -1;
    for (int v = 0; v < p.nlv; v++)
      if (p.lvar[v] == p.pj[q]) a = v;
    if (a < 0) {
      a = p.nlv++;
      p.lvar[a] = p.pj[q];
    }
    for (int v = 0; v < p.nrv; v++)
      if (p.rvar[v] == p.pk[q]) b = v;
    if (b < 0) {
      b = p.nrv++;
      p.rvar[b] = p.pk[q];
    }
    p.pl[q] = a;
    p.pr[q] = b;
  }
  pl->device = device;
  pl->W = p.W;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete pl;
    return fail(MPT_ENODEV, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  }
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  pl->optin = optin;
  // largest k-chunk that fits in shared memory
  size_t smem = 0;
  int kc = 64;
  for (; kc >= 1; kc = kc > 8 ? kc - 8 : kc - 1) {
    p.kc = kc;
    smem = mpt::smem_bytes(p);
    if (smem <= (size_t)optin) break;
  }
  if (kc < 1) {
    delete pl;
    return fail(MPT_EUNSUP, "shared memory budget exceeded");
  }
  // Ensembles (the team kernel, one CTA per trajectory): with enough
  // trajectories to fill every SM twice, size the register budget and the
  // k-chunk for two resident CTAs per SM so that one trajectory's barriers and
  // HBM row loads overlap another's products. MPT_TEAM_MB=1 turns it off.
  p.team_mb = 1;
  {
    int nsm = 0, smem_sm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    pl->nsm = nsm;
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
    pl->smem_sm = smem_sm;
    const char* em = getenv("MPT_TEAM_MB");
    // four 128-thread CTAs per SM for small digit counts (latency bound), two otherwise
    const int want_mb = em ? atoi(em) : (n_traj >= 8 * nsm && p.W <= 20 ? 8 : n_traj >= 4 * nsm && p.W <= 64 ? 4 : n_traj >= 2 * nsm ? 2 : 1);
    const int kc1 = p.kc;
    for (int mb = want_mb >= 8 ? 8 : want_mb >= 4 ? 4 : want_mb; mb >= 2 && p.NP <= 2 && p.team_mb == 1; mb /= 2) {
      const size_t cap = (size_t)smem_sm / mb - 1024;  // 1 KB per CTA is reserved by the runtime
      p.nthreads = mb >= 8 ? 64 : mb >= 4 ? 128 : 256;
      for (int k2 = kc1; k2 >= 1; k2 = k2 > 8 ? k2 - 8 : k2 - 1) {
        p.kc = k2;
        if (mpt::smem_bytes(p) <= cap) {
          p.team_mb = mb;
          smem = mpt::smem_bytes(p);
          break;
        }
      }
    }
    if (p.team_mb == 1) {
      p.kc = kc1;
      p.nthreads = 256;
    }
  }
  pl->smem = smem;
  {
    // team kernel, Cauchy phase: one thread per (pair, balanced window pair) unit
    // (taylor_kernel.cu phase A); more units than threads would be left out
    const int ngb = (2 * p.Lf) / mpt::kR - (p.Lf - 2) / mpt::kR + 1;
    if (p.NP * ((ngb + 1) / 2) > p.nthreads) {
      delete pl;
      return fail(MPT_EUNSUP, "too many product pairs for this precision on the device (pairs x column windows > threads)");
    }
  }
  size_t rows = (size_t)n_traj * dim * (order + 1);
#define ALLOC(ptr, bytes)                                                         \
  do {                                                                            \
    e = cudaMalloc((void**)&(ptr), (bytes));                                      \
    if (e != cudaSuccess) {                                                       \
      mpt_plan_destroy(pl);                                                       \
      return fail(MPT_ECUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e)); \
    }                                                                             \
  } while (0)
  ALLOC(pl->d_cst, sizeof(int32_t) * (size_t)dim * p.RS);
  ALLOC(pl->d_lin, sizeof(int32_t) * (size_t)dim * dim * p.RS);
  ALLOC(pl->d_q, sizeof(int32_t) * (size_t)(nterms > 0 ? nterms : 1) * p.RS);
  ALLOC(pl->d_ctab, sizeof(int32_t) * (size_t)order * p.RS);
  ALLOC(pl->d_coef, sizeof(int32_t) * rows * p.RS);
  ALLOC(pl->d_rinfo, sizeof(int2) * rows);
  ALLOC(pl->d_state, sizeof(int32_t) * (size_t)n_traj * dim * p.RS);
  ALLOC(pl->d_status, sizeof(int32_t) * (size_t)n_traj);
  cudaMemset(pl->d_state, 0, sizeof(int32_t) * (size_t)n_traj * dim * p.RS);
  cudaMemset(pl->d_coef, 0, sizeof(int32_t) * rows * p.RS);
  cudaEventCreate(&pl->ev0);
  cudaEventCreate(&pl->ev1);
  p.cst = pl->d_cst;
  p.lin = pl->d_lin;
  p.q = pl->d_q;
  p.ctab = pl->d_ctab;
  p.coef = pl->d_coef;
  p.rinfo = pl->d_rinfo;
  p.state = pl->d_state;
  p.status = pl->d_status;
  {
    const char* ek = getenv("MPT_KERNEL");
    const char* ec = getenv("MPT_CLUSTER");
    int kernel = ek ? (strcmp(ek, "team") == 0   ? 1
                       : strcmp(ek, "grid") == 0 ? 4
                       : strcmp(ek, "mx") == 0   ? 6
                       : strcmp(ek, "warp") == 0 ? 7
                       : strcmp(ek, "block") == 0 ? 8
                       : strcmp(ek, "cblock") == 0 ? 9
                                                 : 0)
                    : 0;
    int want = ec ? atoi(ec) : (n_traj == 1 ? 16 : 1);
    int rc = choose_kernel(pl, kernel, want < 1 ? 1 : want);
    if (rc) {
      mpt_plan_destroy(pl);
      return rc;
    }
  }
  *out = pl;
  return MPT_OK;
}

int mpt_plan_configure(mpt_plan* pl, int kernel, int cluster) {
  if (!pl || (kernel != 0 && kernel != 1 && kernel != 4 && kernel != 6 && kernel != 7 && kernel != 8 && kernel != 9) || cluster < 1 ||
      cluster > 16)
    return fail(MPT_EINVAL, "bad configuration");
  return choose_kernel(pl, kernel, cluster);
}

int mpt_plan_kernel(const mpt_plan* pl, int* kernel, int* cluster) {
  if (!pl) return MPT_EINVAL;
  if (kernel) *kernel = pl->kernel;
  if (cluster) *cluster = pl->cluster;
  return MPT_OK;
}

int mpt_plan_destroy(mpt_plan* pl) {
  if (!pl) return MPT_OK;
  cudaFree(pl->d_cst);
  cudaFree(pl->d_lin);
  cudaFree(pl->d_q);
  cudaFree(pl->d_ctab);
  cudaFree(pl->d_coef);
  cudaFree(pl->d_rinfo);
  cudaFree(pl->d_state);
  cudaFree(pl->d_rec);
  cudaFree(pl->d_status);
  cudaFree(pl->d_counters);
  cudaFree(pl->d_gscratch);
  cudaFree(pl->d_mxscratch);
  if (pl->ev0) cudaEventDestroy(pl->ev0);
  if (pl->ev1) cudaEventDestroy(pl->ev1);
  delete pl;
  return MPT_OK;
}

int mpt_plan_width(const mpt_plan* pl) { return pl ? pl->W : MPT_EINVAL; }

int mpt_plan_info(const mpt_plan* pl, int* smem_bytes, int* k_chunk, int* threads) {
  if (!pl) return MPT_EINVAL;
  if (smem_bytes) *smem_bytes = (int)(pl->kernel == 4 ? pl->smem_grid : pl->kernel >= 2 ? pl->smem_cluster : pl->smem);
  if (k_chunk && pl->kernel == 4) {
    *k_chunk = pl->grid_kc;
    k_chunk = nullptr;
  }
  if (k_chunk) *k_chunk = pl->p.kc;
  if (threads) *threads = pl->kernel == 7 ? 32 * pl->warp_wpb : pl->kernel == 8 ? 256 : pl->kernel == 9 ? 512 : pl->p.nthreads;
  return MPT_OK;
}

// host values (W digits each) -> device rows (RS stride)
static int upload_rows(int32_t* dst, const int32_t* src, size_t nvals, int W, int RS) {
  std::vector<int32_t> buf(nvals * RS, 0);
  for (size_t v = 0; v < nvals; v++) std::memcpy(&buf[v * RS], src + v * W, sizeof(int32_t) * W);
  CK(cudaMemcpy(dst, buf.data(), sizeof(int32_t) * buf.size(), cudaMemcpyHostToDevice));
  return MPT_OK;
}

static int download_rows(int32_t* dst, const int32_t* src, size_t nvals, int W, int RS) {
  std::vector<int32_t> buf(nvals * RS);
  CK(cudaMemcpy(buf.data(), src, sizeof(int32_t) * buf.size(), cudaMemcpyDeviceToHost));
  for (size_t v = 0; v < nvals; v++) std::memcpy(dst + v * W, &buf[v * RS], sizeof(int32_t) * W);
  return MPT_OK;
}

int mpt_plan_set_constants(mpt_plan* pl, const int32_t* cst, const int32_t* lin, const int32_t* q,
                           const int32_t* ctab) {
  if (!pl || !cst || !lin || !ctab || (pl->p.NT > 0 && !q)) return fail(MPT_EINVAL, "null constant table");
  CK(cudaSetDevice(pl->device));
  const mpt::Params& p = pl->p;
  int rc;
  if ((rc = upload_rows(pl->d_cst, cst, p.D, p.W, p.RS))) return rc;
  if ((rc = upload_rows(pl->d_lin, lin, (size_t)p.D * p.D, p.W, p.RS))) return rc;
  if (p.NT > 0 && (rc = upload_rows(pl->d_q, q, p.NT, p.W, p.RS))) return rc;
  if ((rc = upload_rows(pl->d_ctab, ctab, p.N, p.W, p.RS))) return rc;
  // small-integer coefficients (oracle/fixmodel.c small_int)
  auto small = [&](const int32_t* v, int* out) {
    for (int j = 0; j < p.Lf; j++)
      if (v[j]) return 0;
    if (v[p.Lf] > 4096 || v[p.Lf] < -4096) return 0;
    *out = v[p.Lf];
    return 1;
  };
  mpt::Params& pm = pl->p;
  for (int e = 0; e < p.D * p.D; e++) {
    int val = 0;
    pm.lin_small[e] = small(lin + (size_t)e * p.W, &val);
    pm.lin_int[e] = val;
  }
  for (int r = 0; r < p.NP; r++) pm.pair_round[r] = 0;
  pm.all_q_small = 1;
  for (int t = 0; t < p.NT; t++) {
    int val = 0;
    pm.tq_small[t] = small(q + (size_t)t * p.W, &val);
    pm.tq_int[t] = val;
    if (!pm.tq_small[t]) {
      pm.pair_round[p.tpair[t]] = 1;
      pm.all_q_small = 0;
    }
  }
  for (int t = 0; t < p.NP; t++) pm.tg_used[t] = 1;
  pl->have_constants = true;
  for (int m = 0; m < p.D; m++) {
    pm.tg_used[p.NP + m] = 0;
    for (int j = 0; j < p.D; j++)
      if (!pm.lin_small[m * p.D + j]) pm.tg_used[p.NP + m] = 1;
  }
  return choose_kernel(pl, pl->requested_kernel, pl->requested_cluster);
}

static int ensure_rec(mpt_plan* pl, size_t slots) {
  if (slots <= pl->rec_slots) return MPT_OK;
  cudaFree(pl->d_rec);
  pl->d_rec = nullptr;
  CK(cudaMalloc((void**)&pl->d_rec, sizeof(int32_t) * slots * pl->p.n_traj * pl->p.D * pl->p.RS));
  pl->rec_slots = slots;
  return MPT_OK;
}

static int launch(mpt_plan* pl, int n_steps, int start_step, int stride, cudaStream_t stream, int write_coef = 0) {
  mpt::Params p = pl->p;
  p.write_coef = write_coef;
  if (getenv("MPT_DEBUG")) {
    if (!g_dbg) cudaMalloc((void**)&g_dbg, 8 * 65536);
    cudaMemset(g_dbg, 0, 8 * 65536);
    p.dbg = g_dbg;
  } else {
    p.dbg = nullptr;
  }
  p.n_steps = n_steps;
  p.start_step = start_step;
  p.stride = stride;
  p.rec = pl->d_rec;
  p.counters = pl->counting ? pl->d_counters : nullptr;
  CK(cudaEventRecord(pl->ev0, stream));
  if (pl->kernel == 4) {
    CK(cudaMemsetAsync(pl->d_gscratch, 0, mpt::grid_scratch_bytes(p), stream));
    CK(cudaMemsetAsync(pl->d_status, 0, sizeof(int32_t) * p.n_traj, stream));
    p.gscratch = pl->d_gscratch;
    CK(mpt::launch_grid_kernel(p, pl->grid_blocks, pl->grid_kc, pl->smem_grid, stream));
  } else if (pl->kernel == 6) {
    CK(cudaMemsetAsync(pl->d_status, 0, sizeof(int32_t) * p.n_traj, stream));
    p.gscratch = pl->d_mxscratch;
    CK(mpt::launch_mx_kernel(p, pl->cluster, pl->smem_cluster, stream));
  } else if (pl->kernel == 7) {
    CK(mpt::launch_warp_kernel(p, pl->warp_wpb, stream));
  } else if (pl->kernel == 8) {
    CK(mpt::launch_block_kernel(p, stream));
  } else if (pl->kernel == 9) {
    CK(mpt::launch_cblock_kernel(p, pl->cluster, pl->smem_cluster, stream));
  } else {
    CK(mpt::launch_team_kernel(p, pl->smem, stream));
  }
  CK(cudaEventRecord(pl->ev1, stream));
  return MPT_OK;
}

static int finish(mpt_plan* pl, cudaStream_t stream, int32_t* status) {
  CK(cudaStreamSynchronize(stream));
  CK(cudaGetLastError());
  cudaEventElapsedTime(&pl->last_ms, pl->ev0, pl->ev1);
  if (status) CK(cudaMemcpy(status, pl->d_status, sizeof(int32_t) * pl->p.n_traj, cudaMemcpyDeviceToHost));
  return MPT_OK;
}

int mpt_state_upload(mpt_plan* pl, const int32_t* state0) {
  if (!pl || !state0) return fail(MPT_EINVAL, "null argument");
  CK(cudaSetDevice(pl->device));
  return upload_rows(pl->d_state, state0, (size_t)pl->p.n_traj * pl->p.D, pl->p.W, pl->p.RS);
}

int mpt_state_download(mpt_plan* pl, int32_t* state) {
  if (!pl || !state) return fail(MPT_EINVAL, "null argument");
  CK(cudaSetDevice(pl->device));
  return download_rows(state, pl->d_state, (size_t)pl->p.n_traj * pl->p.D, pl->p.W, pl->p.RS);
}

int mpt_integrate(mpt_plan* pl, const int32_t* state0, int n_steps, int start_step, int stride,
                  int32_t* rec_steps, int32_t* records, int32_t* status) {
  if (!pl || !state0 || !records || !rec_steps) return fail(MPT_EINVAL, "null argument");
  if (!pl->have_constants) return fail(MPT_EINVAL, "constants not set");
  int nrec = mpt_record_count(n_steps, start_step, stride);
  if (nrec < 1 || start_step < 0) return fail(MPT_EINVAL, "invalid step range");
  CK(cudaSetDevice(pl->device));
  int rc;
  if ((rc = ensure_rec(pl, nrec))) return rc;
  if ((rc = mpt_state_upload(pl, state0))) return rc;
  cudaStream_t s = 0;
  if (n_steps > start_step) {
    if ((rc = launch(pl, n_steps, start_step, stride, s))) return rc;
    if ((rc = finish(pl, s, status))) return rc;
  } else if (status) {
    std::memset(status, 0, sizeof(int32_t) * pl->p.n_traj);
  }
  const mpt::Params& p = pl->p;
  size_t per = (size_t)p.n_traj * p.D;
  std::memcpy(records, state0, sizeof(int32_t) * per * p.W);
  if (nrec > 1 && (rc = download_rows(records + per * p.W, pl->d_rec + per * p.RS, per * (nrec - 1), p.W, p.RS)))
    return rc;
  int r = 0;
  rec_steps[r++] = start_step;
  for (int n = start_step + 1; n <= n_steps; n++)
    if (n % stride == 0 || n == n_steps) rec_steps[r++] = n;
  if (status)
    for (int t = 0; t < p.n_traj; t++)
      if (status[t]) return fail(MPT_ERANGE, "fixed-point range exceeded on the device");
  return nrec;
}

int mpt_integrate_device(mpt_plan* pl, int n_steps, void* stream) {
  if (!pl || !pl->have_constants) return fail(MPT_EINVAL, "plan not ready");
  CK(cudaSetDevice(pl->device));
  int rc;
  // records are only written for multiples of `stride`: use a stride beyond n_steps
  if ((rc = ensure_rec(pl, 2))) return rc;
  return launch(pl, n_steps, 0, n_steps + 1, (cudaStream_t)stream);
}

int mpt_compute_jet(mpt_plan* pl, const int32_t* state, int32_t* coef, int32_t* status) {
  if (!pl || !state || !coef) return fail(MPT_EINVAL, "null argument");
  if (!pl->have_constants) return fail(MPT_EINVAL, "constants not set");
  CK(cudaSetDevice(pl->device));
  int rc;
  if ((rc = ensure_rec(pl, 2))) return rc;
  if ((rc = mpt_state_upload(pl, state))) return rc;
  if ((rc = launch(pl, 1, 0, 2, 0, 1))) return rc;
  if ((rc = finish(pl, 0, status))) return rc;
  const mpt::Params& p = pl->p;
  if ((rc = download_rows(coef, pl->d_coef, (size_t)p.n_traj * p.D * (p.N + 1), p.W, p.RS))) return rc;
  if (status)
    for (int t = 0; t < p.n_traj; t++)
      if (status[t]) return fail(MPT_ERANGE, "fixed-point range exceeded on the device");
  return MPT_OK;
}

int mpt_step(mpt_plan* pl, const int32_t* state, int32_t* state_out, int32_t* status) {
  if (!pl || !state || !state_out) return fail(MPT_EINVAL, "null argument");
  CK(cudaSetDevice(pl->device));
  int rc;
  if ((rc = ensure_rec(pl, 2))) return rc;
  if ((rc = mpt_state_upload(pl, state))) return rc;
  if ((rc = launch(pl, 1, 0, 2, 0))) return rc;
  if ((rc = finish(pl, 0, status))) return rc;
  if ((rc = mpt_state_download(pl, state_out))) return rc;
  if (status)
    for (int t = 0; t < pl->p.n_traj; t++)
      if (status[t]) return fail(MPT_ERANGE, "fixed-point range exceeded on the device");
  return MPT_OK;
}

int mpt_debug_read(long long* host, int n) {
  if (!g_dbg) return MPT_EINVAL;
  cudaMemcpy(host, g_dbg, 8 * (size_t)n, cudaMemcpyDeviceToHost);
  return MPT_OK;
}

float mpt_last_kernel_ms(const mpt_plan* pl) {
  if (!pl) return -1.f;
  // the launch may have been asynchronous (mpt_integrate_device): wait for its end event
  if (cudaEventSynchronize(pl->ev1) == cudaSuccess) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, pl->ev0, pl->ev1) == cudaSuccess) return ms;
  }
  cudaGetLastError();
  return pl->last_ms;
}

int mpt_count_macs(mpt_plan* pl, int enable) {
  if (!pl) return fail(MPT_EINVAL, "null plan");
  CK(cudaSetDevice(pl->device));
  if (enable && !pl->d_counters) CK(cudaMalloc((void**)&pl->d_counters, 2 * sizeof(unsigned long long)));
  if (pl->d_counters) CK(cudaMemset(pl->d_counters, 0, 2 * sizeof(unsigned long long)));
  pl->counting = enable != 0;
  return MPT_OK;
}

int mpt_read_macs(mpt_plan* pl, unsigned long long* useful, unsigned long long* executed) {
  if (!pl || !pl->d_counters) return fail(MPT_EINVAL, "counting not enabled");
  unsigned long long h[2];
  CK(cudaMemcpy(h, pl->d_counters, sizeof h, cudaMemcpyDeviceToHost));
  if (useful) *useful = h[0];
  if (executed) *executed = h[1];
  return MPT_OK;
}

int mpt_imad_probe(int device, double* per_second, float* ms_out) {
  if (mpt_device_count() <= 0) return fail(MPT_ENODEV, "no CUDA device available");
  CK(cudaSetDevice(device));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  long long* out = nullptr;
  CK(cudaMalloc((void**)&out, sizeof(long long)));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int threads = 512, blocks = sms * 4, iters = 4096;
  CK(mpt::launch_imad_probe(blocks, threads, 64, out, 0));  // warm-up
  CK(cudaEventRecord(a, 0));
  CK(mpt::launch_imad_probe(blocks, threads, iters, out, 0));
  CK(cudaEventRecord(b, 0));
  CK(cudaEventSynchronize(b));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  double ops = (double)blocks * threads * iters * 64.0;  // 8 unrolled x 8 chains
  if (per_second) *per_second = ops / (ms * 1e-3);
  if (ms_out) *ms_out = ms;
  return MPT_OK;
}

int mpt_l2_flush(int device, size_t bytes) {
  static void* buf = nullptr;
  static size_t have = 0;
  CK(cudaSetDevice(device));
  if (bytes > have) {
    cudaFree(buf);
    buf = nullptr;
    CK(cudaMalloc(&buf, bytes));
    have = bytes;
  }
  CK(cudaMemsetAsync(buf, have & 1, bytes, 0));
  return MPT_OK;
}

}  // extern "C"
