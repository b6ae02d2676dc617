/*
 * oracle/mpfr_ref.c -- CPU restatement of the reference's multiple-precision
 * Taylor hot path, on the reference's own arithmetic backend (MPFR).
 *
 * TEST INFRASTRUCTURE ONLY: called by tests/, by __graft_entry__.smoke() as
 * the checker, and by bench.py's cpu_baseline / --impl reference leg. The
 * product path (paper_1908_09301_b200) never links or calls this file.
 *
 * What it restates (reference = /root/reference/pkg/src/mptaylor):
 *   taylor.py:117 _jet_rows        order loop, frozen evaluation order:
 *                                  constant (i==0 only), linear terms in
 *                                  ascending j, bilinear terms in stored order,
 *                                  then one multiply by inv = div(1, i+1).
 *   reduction.py:93  _fold_chunk    ascending-k fold, one rounding per mul/add,
 *                                  all product pairs fused in one pass.
 *   reduction.py:126 _merge_partials ascending chunk order, empty chunks skipped.
 *   reduction.py:136 _convolve_value serial fold below threshold / 1 chunk,
 *                                  else chunk_bounds partition (reduction.py:84).
 *   taylor.py:168 horner_eval       acc = a[N]; acc = add(a[idx], mul(tau, acc)).
 *   taylor.py:202 integrate         one jet per step, record every stride +
 *                                  final step, absolute stride grid on resume.
 * Every operation is an MPFR call with MPFR_RNDN at the context precision,
 * which is exactly what gmpy2's context methods do for the reference.
 *
 * The chunk loop of one order is run with OpenMP threads (the paper's
 * parallelisation, Fig. 3); each chunk has a single writer and partials are
 * merged in ascending chunk order, so the bits do not depend on the thread
 * count (reduction.py module docstring).
 *
 * Values cross this ABI as (sgn, exp, limbs): value = sgn * M * 2^exp with M
 * the little-endian 64-bit limb integer; sgn in {+1,-1} for nonzero values,
 * 0 for +0 and -2 for -0.
 */
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include "mpfr_min.h"

#define RND MPFR_RNDN

static void import_value(mpfr_ptr x, int32_t sgn, int64_t ex, const uint64_t *limbs, int nl) {
  if (sgn == 0 || sgn == -2) {
    mpfr_set_ui(x, 0, RND);
    if (sgn == -2) mpfr_neg(x, x, RND);
    return;
  }
  mpz_t z;
  __gmpz_init(z);
  __gmpz_import(z, (size_t)nl, -1, 8, 0, 0, limbs);
  mpfr_set_z_2exp(x, z, (mpfr_exp_t)ex, RND); /* exact when M fits the precision */
  if (sgn < 0) mpfr_neg(x, x, RND);
  __gmpz_clear(z);
}

/* returns 0 on success, -1 if the mantissa does not fit nl limbs */
static int export_value(mpfr_srcptr x, int32_t *sgn, int64_t *ex, uint64_t *limbs, int nl) {
  memset(limbs, 0, sizeof(uint64_t) * (size_t)nl);
  if (mpfr_zero_p(x)) {
    *sgn = mpfr_signbit(x) ? -2 : 0;
    *ex = 0;
    return 0;
  }
  mpz_t z;
  __gmpz_init(z);
  mpfr_exp_t e = mpfr_get_z_2exp(z, x);
  int neg = z->_mp_size < 0;
  if (neg) __gmpz_neg(z, z);
  size_t count = (size_t)(z->_mp_size);
  int rc = 0;
  if (count > (size_t)nl) {
    rc = -1;
  } else {
    __gmpz_export(limbs, &count, -1, 8, 0, 0, z);
  }
  *sgn = neg ? -1 : 1;
  *ex = (int64_t)e;
  __gmpz_clear(z);
  return rc;
}

typedef struct {
  int dim, nterms, npairs;
  mpfr_t *constant; /* dim */
  mpfr_t *linear;   /* dim*dim, row m = equation m */
  mpfr_t *tcoef;    /* nterms, grouped by equation in stored order */
  int *teq, *tj, *tk, *tpair;
  int *pj, *pk; /* distinct (j,k) in first-appearance order: systems.py:65 product_pairs */
} sys_t;

static void sys_free(sys_t *s) {
  for (int i = 0; i < s->dim; i++) mpfr_clear(s->constant[i]);
  for (int i = 0; i < s->dim * s->dim; i++) mpfr_clear(s->linear[i]);
  for (int i = 0; i < s->nterms; i++) mpfr_clear(s->tcoef[i]);
  free(s->constant); free(s->linear); free(s->tcoef);
  free(s->teq); free(s->tj); free(s->tk); free(s->tpair); free(s->pj); free(s->pk);
}

/* packed inputs: constants(dim), linear(dim*dim), term coefs(nterms) */
static void sys_build(sys_t *s, int prec, int dim, int nterms, const int32_t *teq,
                      const int32_t *tj, const int32_t *tk, const int32_t *sgn,
                      const int64_t *ex, const uint64_t *limbs, int nl) {
  s->dim = dim;
  s->nterms = nterms;
  s->constant = malloc(sizeof(mpfr_t) * (size_t)dim);
  s->linear = malloc(sizeof(mpfr_t) * (size_t)(dim * dim));
  s->tcoef = malloc(sizeof(mpfr_t) * (size_t)(nterms > 0 ? nterms : 1));
  s->teq = malloc(sizeof(int) * (size_t)(nterms + 1));
  s->tj = malloc(sizeof(int) * (size_t)(nterms + 1));
  s->tk = malloc(sizeof(int) * (size_t)(nterms + 1));
  s->tpair = malloc(sizeof(int) * (size_t)(nterms + 1));
  s->pj = malloc(sizeof(int) * (size_t)(nterms + 1));
  s->pk = malloc(sizeof(int) * (size_t)(nterms + 1));
  int v = 0;
  for (int m = 0; m < dim; m++, v++) {
    mpfr_init2(s->constant[m], prec);
    import_value(s->constant[m], sgn[v], ex[v], limbs + (size_t)v * nl, nl);
  }
  for (int q = 0; q < dim * dim; q++, v++) {
    mpfr_init2(s->linear[q], prec);
    import_value(s->linear[q], sgn[v], ex[v], limbs + (size_t)v * nl, nl);
  }
  s->npairs = 0;
  for (int t = 0; t < nterms; t++, v++) {
    mpfr_init2(s->tcoef[t], prec);
    import_value(s->tcoef[t], sgn[v], ex[v], limbs + (size_t)v * nl, nl);
    s->teq[t] = teq[t];
    s->tj[t] = tj[t];
    s->tk[t] = tk[t];
    int p = -1;
    for (int q = 0; q < s->npairs; q++)
      if (s->pj[q] == tj[t] && s->pk[q] == tk[t]) p = q;
    if (p < 0) {
      p = s->npairs++;
      s->pj[p] = tj[t];
      s->pk[p] = tk[t];
    }
    s->tpair[t] = p;
  }
}

/* reduction.py:84 chunk_bounds */
static void chunk_bounds(int i, int nchunks, int c, int *lo, int *hi) {
  int total = i + 1;
  int base = total / nchunks, rem = total % nchunks;
  *lo = c * base + (c < rem ? c : rem);
  int size = base + (c < rem ? 1 : 0);
  *hi = *lo + size - 1;
}

typedef struct {
  int dim, order, prec;
  mpfr_t *coef; /* dim * (order+1) */
} jet_t;

#define COEF(J, m, i) ((J)->coef[(size_t)(m) * ((J)->order + 1) + (i)])

/* reduction.py:93 _fold_chunk for every pair, k in [lo, hi] */
static void fold_chunk(const sys_t *s, jet_t *J, int i, int lo, int hi, mpfr_t *sums, mpfr_ptr tmp) {
  for (int p = 0; p < s->npairs; p++)
    mpfr_mul(sums[p], COEF(J, s->pj[p], i - lo), COEF(J, s->pk[p], lo), RND);
  for (int k = lo + 1; k <= hi; k++) {
    for (int p = 0; p < s->npairs; p++) {
      mpfr_mul(tmp, COEF(J, s->pj[p], i - k), COEF(J, s->pk[p], k), RND);
      mpfr_add(sums[p], sums[p], tmp, RND);
    }
  }
}

typedef struct {
  int nchunks, threshold, nthreads;
  mpfr_t *part; /* nchunks * npairs */
  mpfr_t *tmp;  /* nchunks */
} red_t;

/* reduction.py:136 _convolve_value */
static void convolve_value(const sys_t *s, jet_t *J, int i, red_t *R, mpfr_t *sums, mpfr_ptr tmp) {
  int c_eff = R->nchunks;
  if (i + 1 < R->threshold || c_eff == 1) {
    fold_chunk(s, J, i, 0, i, sums, tmp);
    return;
  }
  int np = s->npairs;
#pragma omp parallel for schedule(dynamic, 1) num_threads(R->nthreads) if (R->nthreads > 1)
  for (int c = 0; c < c_eff; c++) {
    int lo, hi;
    chunk_bounds(i, c_eff, c, &lo, &hi);
    if (lo <= hi) fold_chunk(s, J, i, lo, hi, R->part + (size_t)c * np, R->tmp[c]);
  }
  int first = 1;
  for (int c = 0; c < c_eff; c++) {
    int lo, hi;
    chunk_bounds(i, c_eff, c, &lo, &hi);
    if (lo > hi) continue;
    for (int p = 0; p < np; p++) {
      if (first)
        mpfr_set(sums[p], R->part[(size_t)c * np + p], RND);
      else
        mpfr_add(sums[p], sums[p], R->part[(size_t)c * np + p], RND);
    }
    first = 0;
  }
}

/* taylor.py:117 _jet_rows; J->coef[m][0] must hold the state */
static void jet_rows(const sys_t *s, jet_t *J, red_t *R, mpfr_t *sums, mpfr_ptr tmp, mpfr_ptr acc,
                     mpfr_ptr inv, mpfr_ptr one) {
  int dim = s->dim;
  for (int i = 0; i < J->order; i++) {
    if (s->npairs) convolve_value(s, J, i, R, sums, tmp);
    mpfr_div_ui(inv, one, (unsigned long)(i + 1), RND);
    for (int m = 0; m < dim; m++) {
      int have = 0;
      if (i == 0) {
        mpfr_set(acc, s->constant[m], RND);
        have = 1;
      }
      for (int j = 0; j < dim; j++) {
        if (have) {
          mpfr_mul(tmp, s->linear[m * dim + j], COEF(J, j, i), RND);
          mpfr_add(acc, acc, tmp, RND);
        } else {
          mpfr_mul(acc, s->linear[m * dim + j], COEF(J, j, i), RND);
          have = 1;
        }
      }
      for (int t = 0; t < s->nterms; t++) {
        if (s->teq[t] != m) continue;
        mpfr_mul(tmp, s->tcoef[t], sums[s->tpair[t]], RND);
        mpfr_add(acc, acc, tmp, RND);
      }
      mpfr_mul(COEF(J, m, i + 1), acc, inv, RND);
    }
  }
}

/* taylor.py:168 horner_eval */
static void horner(jet_t *J, int m, mpfr_srcptr tau, mpfr_ptr out, mpfr_ptr tmp) {
  int n = J->order;
  if (mpfr_zero_p(tau)) {
    mpfr_set(out, COEF(J, m, 0), RND);
    return;
  }
  mpfr_set(out, COEF(J, m, n), RND);
  for (int idx = n - 1; idx >= 0; idx--) {
    mpfr_mul(tmp, tau, out, RND);
    mpfr_add(out, COEF(J, m, idx), tmp, RND);
  }
}

typedef struct {
  sys_t sys;
  jet_t jet;
  red_t red;
  mpfr_t *sums;
  mpfr_t tmp, acc, inv, one, tau;
  mpfr_t *state;
} run_t;

static void run_init(run_t *r, int prec, int dim, int nterms, const int32_t *teq, const int32_t *tj,
                     const int32_t *tk, const int32_t *sgn, const int64_t *ex, const uint64_t *limbs,
                     int nl, int order, int nchunks, int threshold, int nthreads) {
  sys_build(&r->sys, prec, dim, nterms, teq, tj, tk, sgn, ex, limbs, nl);
  r->jet.dim = dim;
  r->jet.order = order;
  r->jet.prec = prec;
  r->jet.coef = malloc(sizeof(mpfr_t) * (size_t)dim * (order + 1));
  for (size_t q = 0; q < (size_t)dim * (order + 1); q++) mpfr_init2(r->jet.coef[q], prec);
  int np = r->sys.npairs > 0 ? r->sys.npairs : 1;
  r->sums = malloc(sizeof(mpfr_t) * np);
  for (int p = 0; p < np; p++) mpfr_init2(r->sums[p], prec);
  r->red.nchunks = nchunks;
  r->red.threshold = threshold;
  r->red.nthreads = nthreads;
  r->red.part = malloc(sizeof(mpfr_t) * (size_t)nchunks * np);
  r->red.tmp = malloc(sizeof(mpfr_t) * (size_t)nchunks);
  for (size_t q = 0; q < (size_t)nchunks * np; q++) mpfr_init2(r->red.part[q], prec);
  for (int c = 0; c < nchunks; c++) mpfr_init2(r->red.tmp[c], prec);
  mpfr_init2(r->tmp, prec);
  mpfr_init2(r->acc, prec);
  mpfr_init2(r->inv, prec);
  mpfr_init2(r->one, prec);
  mpfr_init2(r->tau, prec);
  mpfr_set_ui(r->one, 1, RND);
  r->state = malloc(sizeof(mpfr_t) * dim);
  for (int m = 0; m < dim; m++) mpfr_init2(r->state[m], prec);
}

static void run_free(run_t *r) {
  int np = r->sys.npairs > 0 ? r->sys.npairs : 1;
  for (size_t q = 0; q < (size_t)r->jet.dim * (r->jet.order + 1); q++) mpfr_clear(r->jet.coef[q]);
  for (int p = 0; p < np; p++) mpfr_clear(r->sums[p]);
  for (size_t q = 0; q < (size_t)r->red.nchunks * np; q++) mpfr_clear(r->red.part[q]);
  for (int c = 0; c < r->red.nchunks; c++) mpfr_clear(r->red.tmp[c]);
  for (int m = 0; m < r->jet.dim; m++) mpfr_clear(r->state[m]);
  mpfr_clear(r->tmp); mpfr_clear(r->acc); mpfr_clear(r->inv); mpfr_clear(r->one); mpfr_clear(r->tau);
  free(r->jet.coef); free(r->sums); free(r->red.part); free(r->red.tmp); free(r->state);
  sys_free(&r->sys);
}

const char *ref_mpfr_version(void) { return mpfr_get_version(); }

/*
 * One jet (taylor.py:139 compute_jet). Inputs packed as
 * [constants(dim), linear(dim*dim), term coefs(nterms), state(dim)].
 * Output: dim*(order+1) values, row-major by variable.
 */
int ref_compute_jet(int prec, int dim, int nterms, const int32_t *teq, const int32_t *tj,
                    const int32_t *tk, const int32_t *sgn, const int64_t *ex, const uint64_t *limbs,
                    int nl, int order, int nchunks, int threshold, int nthreads, int32_t *osgn,
                    int64_t *oex, uint64_t *olimbs, int onl) {
  run_t r;
  run_init(&r, prec, dim, nterms, teq, tj, tk, sgn, ex, limbs, nl, order, nchunks, threshold, nthreads);
  int base = dim + dim * dim + nterms;
  for (int m = 0; m < dim; m++)
    import_value(COEF(&r.jet, m, 0), sgn[base + m], ex[base + m], limbs + (size_t)(base + m) * nl, nl);
  jet_rows(&r.sys, &r.jet, &r.red, r.sums, r.tmp, r.acc, r.inv, r.one);
  int rc = 0;
  for (int m = 0; m < dim; m++)
    for (int i = 0; i <= order; i++) {
      size_t o = (size_t)m * (order + 1) + i;
      if (export_value(COEF(&r.jet, m, i), osgn + o, oex + o, olimbs + o * onl, onl)) rc = -1;
    }
  run_free(&r);
  return rc;
}

/*
 * taylor.py:202 integrate. Inputs packed as
 * [constants(dim), linear(dim*dim), term coefs(nterms), state0(dim), tau].
 * Records (step, state) for step start_step, every multiple of stride, and
 * n_steps (taylor.py:195 _record_steps); returns the number of records or a
 * negative error (-1 mantissa overflow, -2 record buffer too small).
 */
int ref_integrate(int prec, int dim, int nterms, const int32_t *teq, const int32_t *tj,
                  const int32_t *tk, const int32_t *sgn, const int64_t *ex, const uint64_t *limbs,
                  int nl, int order, int n_steps, int start_step, int stride, int nchunks,
                  int threshold, int nthreads, int max_rec, int32_t *rec_step, int32_t *osgn,
                  int64_t *oex, uint64_t *olimbs, int onl) {
  run_t r;
  run_init(&r, prec, dim, nterms, teq, tj, tk, sgn, ex, limbs, nl, order, nchunks, threshold, nthreads);
  int base = dim + dim * dim + nterms;
  for (int m = 0; m < dim; m++)
    import_value(r.state[m], sgn[base + m], ex[base + m], limbs + (size_t)(base + m) * nl, nl);
  import_value(r.tau, sgn[base + dim], ex[base + dim], limbs + (size_t)(base + dim) * nl, nl);
  int nrec = 0, rc = 0;
#define RECORD(stepv)                                                                   \
  do {                                                                                  \
    if (nrec >= max_rec) { rc = -2; goto done; }                                        \
    rec_step[nrec] = (stepv);                                                           \
    for (int m = 0; m < dim; m++) {                                                     \
      size_t o = (size_t)nrec * dim + m;                                                \
      if (export_value(r.state[m], osgn + o, oex + o, olimbs + o * onl, onl)) rc = -1;  \
    }                                                                                   \
    nrec++;                                                                             \
  } while (0)
  RECORD(start_step);
  for (int n = start_step + 1; n <= n_steps; n++) {
    for (int m = 0; m < dim; m++) mpfr_set(COEF(&r.jet, m, 0), r.state[m], RND);
    jet_rows(&r.sys, &r.jet, &r.red, r.sums, r.tmp, r.acc, r.inv, r.one);
    for (int m = 0; m < dim; m++) horner(&r.jet, m, r.tau, r.state[m], r.tmp);
    if (n % stride == 0 || n == n_steps) RECORD(n);
  }
done:
  run_free(&r);
  return rc < 0 ? rc : nrec;
}

/* reduction.py:149 convolve / convolve_pair (npairs = 1 or 2 arrays pairs) */
int ref_convolve(int prec, int npairs, int len, const int32_t *sgn, const int64_t *ex,
                 const uint64_t *limbs, int nl, int i, int nchunks, int threshold, int nthreads,
                 int32_t *osgn, int64_t *oex, uint64_t *olimbs, int onl) {
  /* arrays packed as 2*npairs rows of len values: a, b[, c, d] */
  sys_t s;
  memset(&s, 0, sizeof s);
  s.dim = 2 * npairs;
  s.npairs = npairs;
  int pj[2] = {0, 2}, pk[2] = {1, 3};
  s.pj = pj;
  s.pk = pk;
  jet_t J;
  J.dim = 2 * npairs;
  J.order = len - 1;
  J.prec = prec;
  J.coef = malloc(sizeof(mpfr_t) * (size_t)J.dim * len);
  for (int v = 0; v < J.dim * len; v++) {
    mpfr_init2(J.coef[v], prec);
    import_value(J.coef[v], sgn[v], ex[v], limbs + (size_t)v * nl, nl);
  }
  red_t R;
  R.nchunks = nchunks;
  R.threshold = threshold;
  R.nthreads = nthreads;
  R.part = malloc(sizeof(mpfr_t) * (size_t)nchunks * npairs);
  R.tmp = malloc(sizeof(mpfr_t) * (size_t)nchunks);
  for (int q = 0; q < nchunks * npairs; q++) mpfr_init2(R.part[q], prec);
  for (int c = 0; c < nchunks; c++) mpfr_init2(R.tmp[c], prec);
  mpfr_t sums[2], tmp;
  for (int p = 0; p < 2; p++) mpfr_init2(sums[p], prec);
  mpfr_init2(tmp, prec);
  convolve_value(&s, &J, i, &R, sums, tmp);
  int rc = 0;
  for (int p = 0; p < npairs; p++)
    if (export_value(sums[p], osgn + p, oex + p, olimbs + (size_t)p * onl, onl)) rc = -1;
  for (int v = 0; v < J.dim * len; v++) mpfr_clear(J.coef[v]);
  for (int q = 0; q < nchunks * npairs; q++) mpfr_clear(R.part[q]);
  for (int c = 0; c < nchunks; c++) mpfr_clear(R.tmp[c]);
  for (int p = 0; p < 2; p++) mpfr_clear(sums[p]);
  mpfr_clear(tmp);
  free(J.coef); free(R.part); free(R.tmp);
  return rc;
}

/* ---- conversion helpers (mp.py:122 mp_from_decimal, systems.py:90 div(8,3)) ---- */
int mpfr_set_str(mpfr_ptr, const char *, int, mpfr_rnd_t);

/* RN_prec of a decimal literal; 0 ok, -1 parse error */
int ref_from_decimal(int prec, const char *text, int32_t *sgn, int64_t *ex, uint64_t *limbs, int nl) {
  mpfr_t x;
  mpfr_init2(x, prec);
  int bad = mpfr_set_str(x, text, 10, RND);
  int rc = bad ? -1 : export_value(x, sgn, ex, limbs, nl);
  mpfr_clear(x);
  return rc;
}

/* RN_prec(a / b) for exact inputs a, b (packed as 2 values) */
int ref_div(int prec, const int32_t *sgn, const int64_t *ex, const uint64_t *limbs, int nl,
            int32_t *osgn, int64_t *oex, uint64_t *olimbs, int onl) {
  mpfr_t a, b, q;
  mpfr_init2(a, 64 * nl + 64);
  mpfr_init2(b, 64 * nl + 64);
  mpfr_init2(q, prec);
  import_value(a, sgn[0], ex[0], limbs, nl);
  import_value(b, sgn[1], ex[1], limbs + nl, nl);
  mpfr_div(q, a, b, RND);
  int rc = export_value(q, osgn, oex, olimbs, onl);
  mpfr_clear(a); mpfr_clear(b); mpfr_clear(q);
  return rc;
}

/* RN_prec of a binary op on exact inputs: op 0 add, 1 sub, 2 mul */
int ref_binop(int prec, int op, const int32_t *sgn, const int64_t *ex, const uint64_t *limbs, int nl,
              int32_t *osgn, int64_t *oex, uint64_t *olimbs, int onl) {
  mpfr_t a, b, q;
  mpfr_init2(a, 64 * nl + 64);
  mpfr_init2(b, 64 * nl + 64);
  mpfr_init2(q, prec);
  import_value(a, sgn[0], ex[0], limbs, nl);
  import_value(b, sgn[1], ex[1], limbs + nl, nl);
  if (op == 0) mpfr_add(q, a, b, RND);
  else if (op == 1) mpfr_sub(q, a, b, RND);
  else mpfr_mul(q, a, b, RND);
  int rc = export_value(q, osgn, oex, olimbs, onl);
  mpfr_clear(a); mpfr_clear(b); mpfr_clear(q);
  return rc;
}
