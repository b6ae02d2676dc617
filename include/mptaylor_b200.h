/*
 * mptaylor_b200.h -- C ABI of the B200 multiple-precision Taylor engine.
 *
 * Plain pointers and sizes only. Values cross this boundary in the device
 * fixed-point format: each value is W = frac_digits + 1 signed
 * 32-bit digits of radix 2^28, little-endian, value = sum d_j 2^(28 j) *
 * 2^(-28 frac_digits), all digits carrying the sign of the value.
 *
 * Entry points and the reference interface each one replaces
 * (/root/reference/pkg/src/mptaylor):
 *
 *   mpt_plan_create / mpt_plan_set_constants
 *       the per-run setup the reference does in taylor.py:202 integrate
 *       (tau = cfg.tau(ctx) at :234, pairs = system.product_pairs() at :239,
 *       systems.py:65) and in reduction.py:187 SerialReducer / :279 ProcessReducer
 *       construction (the coefficient recurrence's session state).
 *   mpt_integrate            taylor.py:202 integrate  (host buffers in/out; the
 *                            stepping loop :242-253, _jet_rows :117, the Cauchy sums
 *                            reduction.py:149 convolve, horner_eval :168)
 *   mpt_integrate_device     the same on device-resident state (no copies)
 *   mpt_compute_jet          taylor.py:139 compute_jet (one jet per trajectory)
 *   mpt_step                 taylor.py:182 step       (n_steps = 1, no records)
 *
 * All functions return 0 on success and a negative code on failure; the
 * message is available from mpt_last_error(). There is no CPU fallback: if no
 * CUDA device is present every entry point fails with MPT_ENODEV.
 */
#ifndef MPTAYLOR_B200_H
#define MPTAYLOR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPT_OK 0
#define MPT_EINVAL -1     /* bad argument */
#define MPT_ENODEV -2     /* no CUDA device / driver */
#define MPT_ECUDA -3      /* CUDA runtime error */
#define MPT_EUNSUP -4     /* system shape not supported by the device kernel */
#define MPT_ERANGE -5     /* a value left the fixed-point range (status flag) */

typedef struct mpt_plan mpt_plan;

int mpt_version(void);
const char *mpt_last_error(void);
int mpt_device_count(void);

/*
 * dim:          state dimension (<= 4)
 * nterms:       bilinear terms, grouped by equation in stored order
 * term_eq/j/k:  equation index and factor indices (j <= k) of each term
 * frac_digits:  Lf, fractional digits (F = 28 Lf fractional bits)
 * c_shift:      extra digits of the tau/(i+1) table (0 or 1)
 * order:        Taylor order N
 * prec_bits:    reference precision P; the state is rounded to P bits per step
 * n_traj:       independent trajectories integrated by one launch
 * device:       CUDA device ordinal
 */
int mpt_plan_create(mpt_plan **plan, int dim, int nterms, const int32_t *term_eq,
                    const int32_t *term_j, const int32_t *term_k, int frac_digits, int c_shift,
                    int order, int prec_bits, int n_traj, int device);
int mpt_plan_destroy(mpt_plan *plan);

/* Kernel selection (default 0 = automatic):
 *   W <= 34 digits, integer bilinear coefficients, rows fit shared memory
 *                      -> 7 warp kernel (one warp per trajectory; ensembles and small
 *                         single trajectories)
 *   ensembles (>= SMs / 2 trajectories) at 35..58 digits
 *                      -> 8 block kernel (one CTA per trajectory, rows in shared memory)
 *   one trajectory     -> 6 mx (matrix recurrence on a 16-CTA cluster, W <= 120 digits),
 *                         else 4 grid kernel (one trajectory on every SM, rows in L2)
 *   ensembles          -> 1 team kernel (one CTA per trajectory, rows in HBM/L2)
 *   on request         -> 9 cblock kernel (one cluster per trajectory, every CTA keeps all rows
 *                         in shared memory, partial Cauchy sums all-gathered through DSMEM;
 *                         W <= 93 digits)
 * kernel: 0 auto, 1 team, 4 grid, 6 mx, 7 warp, 8 block, 9 cblock; cluster: CTAs per trajectory
 * (2..16) for mx and cblock.
 * Environment overrides at plan creation: MPT_KERNEL=team|grid|mx|warp|block|cblock, MPT_CLUSTER=G,
 * MPT_TEAM_MB=1|2|4|8 (team kernel CTAs per SM; default 8 (64 threads) when n_traj >= 8 x SMs
 * and W <= 20, 4 (128 threads) when n_traj >= 4 x SMs and W <= 64, 2 when n_traj >= 2 x SMs). */
int mpt_plan_configure(mpt_plan *plan, int kernel, int cluster);
int mpt_plan_kernel(const mpt_plan *plan, int *kernel, int *cluster);

/* digits per value (W) */
int mpt_plan_width(const mpt_plan *plan);

/*
 * cst:  dim values          (constant terms c_m)
 * lin:  dim*dim values      (linear matrix, row m = equation m)
 * q:    nterms values       (bilinear coefficients)
 * ctab: order values        (round(tau * 2^(F + 28 c_shift) / (i+1)), i = 0..N-1)
 */
int mpt_plan_set_constants(mpt_plan *plan, const int32_t *cst, const int32_t *lin,
                           const int32_t *q, const int32_t *ctab);

/* number of record slots integrate() fills for (n_steps, start_step, stride) */
int mpt_record_count(int n_steps, int start_step, int stride);

/*
 * state0:   n_traj*dim values (host)
 * records:  host buffer of mpt_record_count(...) * n_traj * dim values;
 *           slot 0 = state0, then every multiple of stride, then n_steps
 * rec_steps: host buffer of mpt_record_count(...) step indices
 * status:   n_traj flags (0 ok, 1 overflow) (host)
 * Returns the number of records written or a negative error.
 */
int mpt_integrate(mpt_plan *plan, const int32_t *state0, int n_steps, int start_step, int stride,
                  int32_t *rec_steps, int32_t *records, int32_t *status);

/* Device-resident variant: state stays in HBM between calls; no records. */
int mpt_state_upload(mpt_plan *plan, const int32_t *state0);
int mpt_state_download(mpt_plan *plan, int32_t *state);
int mpt_integrate_device(mpt_plan *plan, int n_steps, void *stream);

/* one jet per trajectory: coef = n_traj*dim*(order+1) values */
int mpt_compute_jet(mpt_plan *plan, const int32_t *state, int32_t *coef, int32_t *status);

/* one step per trajectory: state_out = n_traj*dim values */
int mpt_step(mpt_plan *plan, const int32_t *state, int32_t *state_out, int32_t *status);

/* device time of the last kernel launch of this plan, milliseconds (CUDA events) */
float mpt_last_kernel_ms(const mpt_plan *plan);

/* dynamic shared memory per CTA and k-chunk chosen for this plan */
int mpt_plan_info(const mpt_plan *plan, int *smem_bytes, int *k_chunk, int *threads);

/* ---- measurement helpers (bench.py roofline; not part of the reference interface) ---- */
/* count limb-MACs in subsequent launches: useful = digit products inside the
   nonzero windows (algorithmic work), executed = issued IMAD.WIDE lanes */
int mpt_count_macs(mpt_plan *plan, int enable);
int mpt_read_macs(mpt_plan *plan, unsigned long long *useful, unsigned long long *executed);
/* measured IMAD.WIDE (s64 += s32*s32) throughput of the whole device, per second */
int mpt_imad_probe(int device, double *imad_per_second, float *ms);
/* write `bytes` of a scratch buffer (L2 flush between timed launches) */
int mpt_l2_flush(int device, size_t bytes);

#ifdef __cplusplus
}
#endif
#endif /* MPTAYLOR_B200_H */
