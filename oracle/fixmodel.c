/*
 * oracle/fixmodel.c -- bit-exact CPU model of the device arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY (tests/ and smoke() use it as the checker; the
 * product never links it). It restates, in plain C with exact __int128
 * column sums, the fixed-point algorithm that the sm_100a kernel
 * (paper_1908_09301_b200/csrc/taylor_kernel.cu) implements, so that every
 * coefficient the GPU produces can be compared bit for bit. DESIGN.md §3
 * is the normative description; in short:
 *
 *   digit radix B = 2^28; a value is X * 2^-F, F = 28*Lf, X = sum d_j B^j,
 *   j = 0..Lf, signed digits with |d_j| < B all carrying the sign of X.
 *   Coefficients are tau-scaled (a~_i = a_i tau^i), so the state update is
 *   the exact sum of the coefficient rows.
 *
 *   tprod(A, C, T) = sum_{p+q >= T} a_p c_q B^(p+q-T)   (truncated product)
 *   rnd(V)         = floor((V + B^2/2) / B^2)          (two guard digits)
 *
 *   order i:  V_p  = sum_k tprod(coef[j_p][i-k], coef[k_p][k], Lf-2)   (exact)
 *             U_m  = rnd( [i==0] cst_m B^2 + sum_j tprod(lin[m][j], coef[j][i], Lf-2)
 *                         + sum_t Q_t )
 *             Q_t  = q_t * V_{p_t}                 if q_t is a small integer
 *                    tprod(q_t, rnd(V_{p_t}), Lf-2) otherwise
 *             coef[m][i+1] = rnd( tprod(U_m, Ctab[i], Lf+sc-2) ),
 *   Ctab[i] = round(tau * 2^(F + 28 sc) / (i+1)) computed on the host.
 *   state'[m] = RN_P( sum_i coef[m][i] )  (exact sum, then ties-to-even
 *                 rounding to the reference precision P)
 *
 * Terms are grouped by equation in stored order like the reference's
 * systems.py:32 QuadraticODESystem; pairs are distinct (j,k) in first
 * appearance order (systems.py:65 product_pairs).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define RADIX_BITS 28
#define RADIX ((int64_t)1 << RADIX_BITS)

typedef __int128 i128;

typedef struct {
  int D, NT, NP, Lf, sc, order;
  int variant; /* 0: per-order C-product recurrence, 1: matrix recurrence (jet_mx) */
  const int32_t *cst;  /* D x W */
  const int32_t *lin;  /* D x D x W */
  const int32_t *q;    /* NT x W */
  const int32_t *ctab; /* order x W */
  int teq[64], tj[64], tk[64], tpair[64], pj[64], pk[64];
} model_t;

#define W(M) ((M)->Lf + 1)

/* columns c in [T, T+ncols): out[c-T] += sum_{p+q=c} a_p b_q */
static void tprod_acc(const int32_t *a, const int32_t *b, int L, int T, i128 *col, int ncols) {
  for (int p = 0; p < L; p++) {
    if (!a[p]) continue;
    int q0 = T - p;
    if (q0 < 0) q0 = 0;
    for (int q = q0; q < L; q++) {
      int c = p + q - T;
      if (c >= ncols) break;
      col[c] += (i128)((int64_t)a[p] * (int64_t)b[q]);
    }
  }
}

/* tprod_acc for operands of different lengths */
static void tprod_acc2(const int32_t *a, int La, const int32_t *b, int Lb, int T, i128 *col, int ncols) {
  for (int p = 0; p < La; p++) {
    if (!a[p]) continue;
    int q0 = T - p;
    if (q0 < 0) q0 = 0;
    for (int q = q0; q < Lb; q++) {
      int c = p + q - T;
      if (c >= ncols) break;
      col[c] += (i128)((int64_t)a[p] * (int64_t)b[q]);
    }
  }
}

/* V = sum col[c] B^c (exact), return digits of rnd(V) = floor((V + B^2/2)/B^2) in out[0..Lf];
   returns 1 on overflow (result does not fit Lf+1 digits) */
static int round_cols_canon(const i128 *col, int ncols, int Lf, int32_t *out) {
  /* normalize to digits in [0, B) with floor carries, keep the top carry */
  i128 carry = 0;
  int64_t dig[4096 + 8];
  for (int c = 0; c < ncols; c++) {
    i128 v = col[c] + carry;
    i128 d = v & (RADIX - 1);
    carry = (v - d) >> RADIX_BITS; /* exact floor division */
    dig[c] = (int64_t)d;
  }
  /* add B^2/2: digit 1 gets B/2 */
  i128 v = (i128)dig[1] + (RADIX / 2);
  int64_t cin = (int64_t)(v >> RADIX_BITS);
  dig[1] = (int64_t)(v & (RADIX - 1));
  for (int c = 2; c < ncols && cin; c++) {
    v = (i128)dig[c] + cin;
    cin = (int64_t)(v >> RADIX_BITS);
    dig[c] = (int64_t)(v & (RADIX - 1));
  }
  carry += cin;
  /* result digits = dig[2..], value = sum dig[2+j] B^j + carry B^(ncols-2) (two's-complement-like) */
  int nres = ncols - 2;
  /* build signed result: if carry < 0 the number is negative; convert to sign-magnitude */
  int neg = carry < 0;
  int32_t mag[4096 + 8];
  if (!neg) {
    for (int j = 0; j < nres; j++) mag[j] = (int32_t)dig[2 + j];
    if (carry != 0) return 1;
  } else {
    /* magnitude = -(value) = B^nres * (-carry) - sum dig B^j */
    int64_t borrow = 0;
    for (int j = 0; j < nres; j++) {
      int64_t t = -dig[2 + j] - borrow;
      if (t < 0) {
        t += RADIX;
        borrow = 1;
      } else {
        borrow = 0;
      }
      mag[j] = (int32_t)t;
    }
    /* remaining high part: -carry - borrow must be 0 */
    if (-carry - borrow != 0) return 1;
  }
  for (int j = nres; j <= Lf; j++) mag[j] = 0;
  for (int j = Lf + 1; j < nres; j++)
    if (mag[j]) return 1;
  for (int j = 0; j <= Lf; j++) out[j] = neg ? -mag[j] : mag[j];
  return 0;
}

/* The per-order rounding of the recurrence: digits of rnd(V) in the device's
   balanced semi-normal form (mpt_device.cuh warp_snf_t). B/2 is added to
   column 1; three rounds of "every column below the top one (index Lf+2)
   splits into a balanced digit in [-B/2, B/2) and the carry round(v/B), which
   moves one column up; the top column absorbs" leave digits in [-B/2-1, B/2];
   digit 2 is corrected by floor((d_0 + d_1 B) / B^2) and digits 2..Lf+2 are
   the result. Returns 1 on overflow (|top digit| >= B). */
static int round_cols(const i128 *col, int ncols, int Lf, int32_t *out) {
  i128 v[4096 + 8];
  const int topc = Lf + 2;
  for (int c = 0; c <= topc; c++) v[c] = c < ncols ? col[c] : 0;
  for (int c = ncols - 1; c > topc; c--) v[topc] += col[c] << (RADIX_BITS * (c - topc));
  v[1] += RADIX / 2;
  for (int r = 0; r < 3; r++) {
    i128 cin = 0;
    for (int c = 0; c < topc; c++) {
      i128 h = (v[c] + RADIX / 2) >> RADIX_BITS;
      v[c] = v[c] - h * RADIX + cin;
      cin = h;
    }
    v[topc] += cin;
  }
  i128 low = v[0] + v[1] * RADIX;
  v[2] += low < 0 ? -1 : (low >= (i128)RADIX * RADIX ? 1 : 0);
  for (int j = 0; j <= Lf; j++) out[j] = (int32_t)v[2 + j];
  return (v[topc] >= RADIX || v[topc] <= -RADIX) ? 1 : 0;
}

/* Rounding of the matrix recurrence (variant 1): digits of
 *     R = floor((V + B^2/2) / B^2),   V = sum_c col[c] B^c   (exact)
 * in the UNIQUE balanced form: R = sum_{j<Wout-1} e_j B^j + e_top B^(Wout-1)
 * with every e_j (top included) in [-B/2, B/2). Unlike round_cols the result
 * depends on the value V only, not on how it is split over the columns, so a
 * device that folds partial column sums differently still agrees bit for bit.
 * Small values of either sign keep leading zero digits. Returns 1 on overflow. */
static int round_bnf(const i128 *col, int ncols, int Wout, int32_t *out) {
  int64_t dig[4096 + 16];
  i128 carry = 0;
  for (int c = 0; c < ncols; c++) {
    i128 v = col[c] + carry + (c == 1 ? (RADIX / 2) : 0);
    i128 d = v & (RADIX - 1);
    carry = (v - d) >> RADIX_BITS;
    dig[c] = (int64_t)d;
  }
  for (int c = ncols; c < Wout + 2; c++) {
    i128 v = carry;
    i128 d = v & (RADIX - 1);
    carry = (v - d) >> RADIX_BITS;
    dig[c] = (int64_t)d;
  }
  const int n = ncols > Wout + 2 ? ncols : Wout + 2;
  /* everything above the top digit column (Wout+1) must vanish in two's complement */
  int ovf = 0;
  i128 hi = carry;
  for (int c = n - 1; c > Wout + 1; c--) {
    hi = hi * RADIX + dig[c];
    if (hi > ((i128)1 << 40) || hi < -((i128)1 << 40)) ovf = 1;
  }
  int t = 0;
  for (int j = 0; j < Wout - 1; j++) {
    int64_t x = dig[2 + j] + t;
    if (x >= RADIX / 2) {
      x -= RADIX;
      t = 1;
    } else {
      t = 0;
    }
    out[j] = (int32_t)x;
  }
  i128 top = (i128)dig[Wout + 1] + t + hi * RADIX;
  if (top >= RADIX / 2 || top < -(RADIX / 2)) ovf = 1;
  out[Wout - 1] = (int32_t)top;
  return ovf;
}

static int build(model_t *M, int D, int NT, const int32_t *teq, const int32_t *tj, const int32_t *tk) {
  if (D > 16 || NT > 64) return -3;
  M->D = D;
  M->NT = NT;
  M->NP = 0;
  for (int t = 0; t < NT; t++) {
    M->teq[t] = teq[t];
    M->tj[t] = tj[t];
    M->tk[t] = tk[t];
    int p = -1;
    for (int r = 0; r < M->NP; r++)
      if (M->pj[r] == tj[t] && M->pk[r] == tk[t]) p = r;
    if (p < 0) {
      p = M->NP++;
      M->pj[p] = tj[t];
      M->pk[p] = tk[t];
    }
    M->tpair[t] = p;
  }
  return 0;
}

/* a constant is a "small integer" when only its integer digit (index Lf) is
   nonzero and |d_Lf| <= 4096; bilinear terms with such coefficients are
   applied to the exact Cauchy column sum (no intermediate rounding) */
static int small_int(const int32_t *v, int Lf, int64_t *out) {
  for (int j = 0; j < Lf; j++)
    if (v[j]) return 0;
  if (v[Lf] > 4096 || v[Lf] < -4096) return 0;
  *out = v[Lf];
  return 1;
}

/* coef: D x (order+1) x W, coef[m][0] set by caller */
static int jet(const model_t *M, int32_t *coef) {
  int Lf = M->Lf, L = Lf + 1, Wd = W(M), D = M->D, N = M->order;
  int ncols = Lf + 3; /* columns [Lf-2, 2Lf] */
  i128 *col = malloc(sizeof(i128) * (size_t)(ncols + 2));
  i128 *V = malloc(sizeof(i128) * (size_t)(M->NP + 1) * ncols);
  int32_t *S = malloc(sizeof(int32_t) * (size_t)(M->NP + 1) * Wd);
  int32_t *U = malloc(sizeof(int32_t) * (size_t)D * Wd);
  int64_t qint[64];
  int qsmall[64];
  for (int t = 0; t < M->NT; t++) qsmall[t] = small_int(M->q + (size_t)t * Wd, Lf, &qint[t]);
  int rc = 0;
#define CO(m, i) (coef + ((size_t)(m) * (N + 1) + (i)) * Wd)
  for (int i = 0; i < N && !rc; i++) {
    for (int p = 0; p < M->NP; p++) {
      i128 *vp = V + (size_t)p * ncols;
      memset(vp, 0, sizeof(i128) * ncols);
      for (int k = 0; k <= i; k++) tprod_acc(CO(M->pj[p], i - k), CO(M->pk[p], k), L, Lf - 2, vp, ncols);
      int need = 0;
      for (int t = 0; t < M->NT; t++)
        if (M->tpair[t] == p && !qsmall[t]) need = 1;
      if (need && round_cols(vp, ncols, Lf, S + (size_t)p * Wd)) rc = 1;
    }
    for (int m = 0; m < D; m++) {
      memset(col, 0, sizeof(i128) * ncols);
      if (i == 0)
        for (int j = 0; j <= Lf; j++) col[2 + j] += (i128)M->cst[(size_t)m * Wd + j];
      for (int j = 0; j < D; j++) tprod_acc(M->lin + ((size_t)m * D + j) * Wd, CO(j, i), L, Lf - 2, col, ncols);
      for (int t = 0; t < M->NT; t++) {
        if (M->teq[t] != m) continue;
        if (qsmall[t]) {
          const i128 *vp = V + (size_t)M->tpair[t] * ncols;
          for (int c = 0; c < ncols; c++) col[c] += (i128)qint[t] * vp[c];
        } else {
          tprod_acc(M->q + (size_t)t * Wd, S + (size_t)M->tpair[t] * Wd, L, Lf - 2, col, ncols);
        }
      }
      if (round_cols(col, ncols, Lf, U + (size_t)m * Wd)) rc = 1;
    }
    for (int m = 0; m < D; m++) {
      memset(col, 0, sizeof(i128) * ncols);
      tprod_acc(U + (size_t)m * Wd, M->ctab + (size_t)i * Wd, L, Lf + M->sc - 2, col, ncols);
      if (round_cols(col, ncols, Lf, CO(m, i + 1))) rc = 1;
    }
  }
  free(col);
  free(V);
  free(S);
  free(U);
  return rc;
}

/* ---------------------------------------------------------------------------
 * Matrix recurrence (variant 1; paper_1908_09301_b200/csrc/taylor_mx.cu).
 * Same quantities, reassociated so that one order costs one product stage and
 * one rounding on the critical path. With a~_{i+1} = C_i U_i the next
 * numerator is linear in U_i except for the Cauchy sums; the Cauchy sum of
 * order j = i+1 is split into its lag-1 terms (rows j-1 and 1, computed next
 * to the recurrence) and the rest L'(j) (rows 2..j-2, computed ahead by the
 * bulk CTAs, owner(k) = 1 + (k-1) mod Gb):
 *
 *   U_j^m = rnd( sum_{j'} tprod(U_i^{j'}, K_i^{m,j'}, Lf+sc-2)
 *               + sum_{t in m} q_t [ lag_t(j) + sum_o split1(P_{o,t}(j)) ] )
 *   K_i^{m,j'} = rnd_{Lf+2 digits}( tprod(S^{m,j'}, C_i, Lf-2) )  (keeps the sc digits of C_i)
 *   S^{m,j'} = bnf( lin[m][j'] + sum_{t in m, j_t=j'} q_t a~^{k_t}_0 + sum_{t in m, k_t=j'} q_t a~^{j_t}_0 )
 *   lag_t(2) = tprod(a~^a_1, a~^b_1),  lag_t(j>=3) = tprod(a~^a_{j-1}, a~^b_1) + tprod(a~^a_1, a~^b_{j-1})
 *   P_{o,t}(j) = sum_{k in [2, j-2], own_j(k) = o} tprod(a~^a_{j-k}, a~^b_k, Lf-2)       (exact)
 *                own_j(k) = owner(k) for k > 2, own_j(2) = owner(j-2) (the newest row's owner)
 *   split1(P)[c] = (P_c mod B) + floor(P_{c-1} / B)   (one carry step, a function of P only)
 *   a~^m_{i+1} = rnd( tprod(U_i^m, C_i, Lf+sc-2) )
 *   U_0 = rnd( cst B^2 + sum_j tprod(lin[m][j], bnf(a~_0^j)) + sum_t q_t tprod(bnf(a~_0^a), bnf(a~_0^b)) )
 *
 * rnd = round_cols applied to EXACT column sums (the device forms them in
 * int64 without folds: every operand digit is balanced or semi-normal), so
 * the rounding is deterministic; bnf = value-exact balanced digits (drop 0).
 * Requires small-integer bilinear coefficients.
 */
static int bnf_exact(const i128 *val, int n, int Wout, int32_t *out) {
  /* balanced digits of V = sum val[c] B^c (no rounding): round_bnf with the two
     guard columns zero and the rounding half cancelled */
  i128 col[4096 + 8];
  col[0] = -(RADIX / 2);
  col[1] = 0;
  for (int c = 0; c < n; c++) col[2 + c] = val[c];
  return round_bnf(col, n + 2, Wout, out);
}

static void split1(const i128 *P, int ncols, i128 *acc, int64_t mult) {
  i128 prev = 0;
  for (int c = 0; c < ncols; c++) {
    i128 lo = P[c] & (RADIX - 1);
    i128 hi_prev = prev >> RADIX_BITS; /* floor */
    acc[c] += (i128)mult * (lo + hi_prev);
    prev = P[c];
  }
}

static int mx_bulk = 15;
void fix_set_bulk(int Gb) { mx_bulk = Gb < 1 ? 1 : Gb; }

static int jet_mx(const model_t *M, int32_t *coef) {
  int Lf = M->Lf, L = Lf + 1, Wd = W(M), D = M->D, N = M->order, sc = M->sc, Gb = mx_bulk;
  int ncols = Lf + 4, KW = Wd + 1;
  int64_t qint[64];
  for (int t = 0; t < M->NT; t++)
    if (!small_int(M->q + (size_t)t * Wd, Lf, &qint[t])) return -5;
  i128 *col = malloc(sizeof(i128) * (size_t)(ncols + 2));
  i128 *P = malloc(sizeof(i128) * (size_t)(ncols + 2));
  int32_t *SB = malloc(sizeof(int32_t) * (size_t)D * Wd);
  int32_t *S = calloc((size_t)D * D * Wd, sizeof(int32_t));
  int32_t *K = malloc(sizeof(int32_t) * (size_t)D * D * KW);
  int32_t *U = malloc(sizeof(int32_t) * (size_t)D * Wd);
  int32_t *U2 = malloc(sizeof(int32_t) * (size_t)D * Wd);
  int snz[256];
  i128 acc[4096 + 8];
  int rc = 0;
#define CO(m, i) (coef + ((size_t)(m) * (N + 1) + (i)) * Wd)
  for (int m = 0; m < D && !rc; m++) {
    for (int d = 0; d <= Lf; d++) acc[d] = CO(m, 0)[d];
    if (bnf_exact(acc, Wd, Wd, SB + (size_t)m * Wd)) rc = 1;
  }
  for (int m = 0; m < D && !rc; m++)
    for (int j = 0; j < D && !rc; j++) {
      for (int d = 0; d <= Lf; d++) acc[d] = M->lin[((size_t)m * D + j) * Wd + d];
      for (int t = 0; t < M->NT; t++) {
        if (M->teq[t] != m) continue;
        if (M->tj[t] == j)
          for (int d = 0; d <= Lf; d++) acc[d] += (i128)qint[t] * CO(M->tk[t], 0)[d];
        if (M->tk[t] == j)
          for (int d = 0; d <= Lf; d++) acc[d] += (i128)qint[t] * CO(M->tj[t], 0)[d];
      }
      int32_t *s = S + ((size_t)m * D + j) * Wd;
      if (bnf_exact(acc, Wd, Wd, s)) rc = 1;
      snz[m * D + j] = 0;
      for (int d = 0; d <= Lf; d++) snz[m * D + j] |= s[d] != 0;
    }
  for (int m = 0; m < D && !rc; m++) {
    memset(col, 0, sizeof(i128) * ncols);
    for (int j = 0; j <= Lf; j++) col[2 + j] += (i128)M->cst[(size_t)m * Wd + j];
    for (int j = 0; j < D; j++) tprod_acc(M->lin + ((size_t)m * D + j) * Wd, SB + (size_t)j * Wd, L, Lf - 2, col, ncols);
    for (int t = 0; t < M->NT; t++) {
      if (M->teq[t] != m) continue;
      memset(P, 0, sizeof(i128) * ncols);
      tprod_acc(SB + (size_t)M->tj[t] * Wd, SB + (size_t)M->tk[t] * Wd, L, Lf - 2, P, ncols);
      for (int c = 0; c < ncols; c++) col[c] += (i128)qint[t] * P[c];
    }
    if (round_cols(col, ncols, Lf, U + (size_t)m * Wd)) rc = 1;
  }
  for (int i = 0; i < N && !rc; i++) {
    const int32_t *C = M->ctab + (size_t)i * Wd;
    for (int m = 0; m < D; m++) {
      memset(col, 0, sizeof(i128) * ncols);
      tprod_acc(U + (size_t)m * Wd, C, L, Lf + sc - 2, col, ncols);
      if (round_cols(col, ncols, Lf, CO(m, i + 1))) rc = 1;
    }
    if (i + 1 >= N) break;
    for (int e = 0; e < D * D; e++) {
      if (!snz[e]) continue;
      memset(col, 0, sizeof(i128) * ncols);
      tprod_acc(S + (size_t)e * Wd, C, L, Lf - 2, col, ncols);
      if (round_cols(col, ncols, Lf + 1, K + (size_t)e * KW)) rc = 1;
    }
    const int j = i + 1;
    for (int m = 0; m < D; m++) {
      memset(col, 0, sizeof(i128) * ncols);
      for (int jj = 0; jj < D; jj++)
        if (snz[m * D + jj])
          tprod_acc2(U + (size_t)jj * Wd, L, K + ((size_t)m * D + jj) * KW, KW, Lf + sc - 2, col, ncols);
      for (int t = 0; t < M->NT; t++) {
        if (M->teq[t] != m) continue;
        const int a = M->tj[t], b = M->tk[t];
        memset(P, 0, sizeof(i128) * ncols);
        if (j == 2) tprod_acc(CO(a, 1), CO(b, 1), L, Lf - 2, P, ncols);
        if (j >= 3) {
          tprod_acc(CO(a, j - 1), CO(b, 1), L, Lf - 2, P, ncols);
          tprod_acc(CO(a, 1), CO(b, j - 1), L, Lf - 2, P, ncols);
        }
        for (int c = 0; c < ncols; c++) col[c] += (i128)qint[t] * P[c];
        for (int o = 1; o <= Gb; o++) {
          memset(P, 0, sizeof(i128) * ncols);
          int any = 0;
          for (int k = 2; k <= j - 2; k++) {
            /* owner(k), except that the k = 2 term goes with the newest row's owner(j-2) */
            const int ok = k == 2 ? 1 + (j - 3) % Gb : 1 + (k - 1) % Gb;
            if (ok != o) continue;
            tprod_acc(CO(a, j - k), CO(b, k), L, Lf - 2, P, ncols);
            any = 1;
          }
          if (any) split1(P, ncols, col, qint[t]);
        }
      }
      if (round_cols(col, ncols, Lf, U2 + (size_t)m * Wd)) rc = 1;
    }
    memcpy(U, U2, sizeof(int32_t) * (size_t)D * Wd);
  }
#undef CO
  free(col);
  free(P);
  free(SB);
  free(S);
  free(K);
  free(U);
  free(U2);
  return rc;
}

/* ---------------------------------------------------------------------------
 * Value-exact recurrence (variant 2; paper_1908_09301_b200/csrc/taylor_lx.cu).
 *
 * The matrix form of variant 1, but every rounding is a function of the VALUE
 * of an exact column sum only, so the device may partition, fold and sum its
 * partial products in any order and still agree bit for bit:
 *
 *   sd(R)  = the signed-digit recoding of the two's-complement radix-B digits
 *            r_j of R:  e_j = r_j - B t_j + t_{j-1},  t_j = [r_j >= B/2]
 *            (digits in [-B/2, B/2]; unique for a value)
 *   rndb(V) = sd( floor((V + B^2/2) / B^2) ),  V = sum_c col[c] B^c exact
 *
 * Per step (a~_0 = the state, canonical digits):
 *   SB^j     = sd(a~_0^j),  Cb_i = sd(C_i)
 *   S^{m,j}  = sd( linN[m][j] + sum_{t in m, j_t = j} q_t SB^{k_t} + sum_{t in m, k_t = j} q_t SB^{j_t} )
 *              (linN = the linear coefficients that are not small integers)
 *   U_0^m    = rndb( cst_m B^2 + sum_j tprod(lin[m][j], SB^j) + sum_t q_t tprod(SB^{j_t}, SB^{k_t}) )
 *   order i: X^j      = tprod(U_i^j, Cb_i, Lf+sc-2)                        (exact columns)
 *            a~^m_{i+1} = rndb(X^m)
 *            K^{m,j}  = rndb_{W+1}( tprod(S^{m,j}, Cb_i, Lf-2) )           (same scale as C)
 *            U_{i+1}^m = rndb( sum_j linI[m][j] X^j + sum_{S^{m,j} structural} tprod(U_i^j, K^{m,j}, Lf+sc-2)
 *                               + sum_{t in m} q_t [ lag_t(i+1) + L'_t(i+1) ] )
 *            lag_t(2) = tprod(a~^a_1, a~^b_1);  lag_t(j>=3) = tprod(a~^a_{j-1}, a~^b_1) + tprod(a~^a_1, a~^b_{j-1})
 *            L'_t(j)  = sum_{k=2}^{j-2} tprod(a~^a_{j-k}, a~^b_k)
 * (tprod without a T argument: T = Lf-2.) linI = the small-integer linear
 * coefficients; they multiply the exact X columns. Requires small-integer
 * bilinear coefficients.
 */

/* digits of R = floor((V + [half] B^drop/2) / B^drop), V = sum col[c] B^c, in
   the sd recoding, Wout digits; returns 1 when R does not fit Wout sd digits */
static int sd_cols(const i128 *col, int ncols, int drop, int half, int Wout, int32_t *out) {
  const int n = (ncols > Wout + drop ? ncols : Wout + drop) + 6;
  int64_t r[4096 + 32];
  i128 carry = 0;
  for (int c = 0; c < n; c++) {
    i128 v = carry + (c < ncols ? col[c] : 0);
    if (half && drop > 0 && c == drop - 1) v += RADIX / 2;
    i128 d = v & (RADIX - 1);
    carry = (v - d) >> RADIX_BITS;
    r[c] = (int64_t)d;
  }
  if (carry != 0 && carry != -1) return 1;
  const int nr = n - drop;
  int t_prev = 0, ovf = 0;
  for (int j = 0; j < nr; j++) {
    const int64_t rj = r[j + drop];
    const int t = rj >= RADIX / 2;
    const int64_t e = rj - (t ? RADIX : 0) + t_prev;
    t_prev = t;
    if (j < Wout) out[j] = (int32_t)e;
    else if (e != 0) ovf = 1;
  }
  /* past digit n the digits are the sign extension: 0 (carry 0) or B-1 (carry -1) */
  if ((carry == 0 && t_prev != 0) || (carry == -1 && t_prev != 1)) ovf = 1;
  return ovf;
}

static int rndb(const i128 *col, int ncols, int Wout, int32_t *out) { return sd_cols(col, ncols, 2, 1, Wout, out); }

static int jet_lx(const model_t *M, int32_t *coef) {
  int Lf = M->Lf, L = Lf + 1, Wd = W(M), D = M->D, N = M->order, sc = M->sc;
  int ncols = Lf + 4, KW = Wd + 1;
  int64_t qint[64], linI[64];
  int linS[64];
  for (int t = 0; t < M->NT; t++)
    if (!small_int(M->q + (size_t)t * Wd, Lf, &qint[t])) return -5;
  for (int e = 0; e < D * D; e++) {
    linS[e] = small_int(M->lin + (size_t)e * Wd, Lf, &linI[e]);
    if (!linS[e]) linI[e] = 0;
  }
  i128 *col = malloc(sizeof(i128) * (size_t)(ncols + 8));
  i128 *X = malloc(sizeof(i128) * (size_t)D * (ncols + 8));
  int32_t *SB = malloc(sizeof(int32_t) * (size_t)D * Wd);
  int32_t *S = calloc((size_t)D * D * Wd, sizeof(int32_t));
  int32_t *K = malloc(sizeof(int32_t) * (size_t)D * D * KW);
  int32_t *Cb = malloc(sizeof(int32_t) * (size_t)(N > 0 ? N : 1) * Wd);
  int32_t *U = malloc(sizeof(int32_t) * (size_t)D * Wd);
  int32_t *U2 = malloc(sizeof(int32_t) * (size_t)D * Wd);
  int snz[256];
  i128 acc[4096 + 8];
  int rc = 0;
#define CO(m, i) (coef + ((size_t)(m) * (N + 1) + (i)) * Wd)
  for (int m = 0; m < D && !rc; m++) {
    for (int d = 0; d <= Lf; d++) acc[d] = CO(m, 0)[d];
    if (sd_cols(acc, Wd, 0, 0, Wd, SB + (size_t)m * Wd)) rc = 1;
  }
  for (int i = 0; i < N && !rc; i++) {
    for (int d = 0; d <= Lf; d++) acc[d] = M->ctab[(size_t)i * Wd + d];
    if (sd_cols(acc, Wd, 0, 0, Wd, Cb + (size_t)i * Wd)) rc = 1;
  }
  for (int m = 0; m < D && !rc; m++)
    for (int j = 0; j < D && !rc; j++) {
      int any = !linS[m * D + j];
      for (int d = 0; d <= Lf; d++) acc[d] = linS[m * D + j] ? 0 : M->lin[((size_t)m * D + j) * Wd + d];
      for (int t = 0; t < M->NT; t++) {
        if (M->teq[t] != m) continue;
        if (M->tj[t] == j) {
          any = 1;
          for (int d = 0; d <= Lf; d++) acc[d] += (i128)qint[t] * SB[(size_t)M->tk[t] * Wd + d];
        }
        if (M->tk[t] == j) {
          any = 1;
          for (int d = 0; d <= Lf; d++) acc[d] += (i128)qint[t] * SB[(size_t)M->tj[t] * Wd + d];
        }
      }
      snz[m * D + j] = any;
      if (sd_cols(acc, Wd, 0, 0, Wd, S + ((size_t)m * D + j) * Wd)) rc = 1;
    }
  for (int m = 0; m < D && !rc; m++) {
    memset(col, 0, sizeof(i128) * ncols);
    for (int j = 0; j <= Lf; j++) col[2 + j] += (i128)M->cst[(size_t)m * Wd + j];
    for (int j = 0; j < D; j++) tprod_acc(M->lin + ((size_t)m * D + j) * Wd, SB + (size_t)j * Wd, L, Lf - 2, col, ncols);
    for (int t = 0; t < M->NT; t++) {
      if (M->teq[t] != m) continue;
      memset(acc, 0, sizeof(i128) * ncols);
      tprod_acc(SB + (size_t)M->tj[t] * Wd, SB + (size_t)M->tk[t] * Wd, L, Lf - 2, acc, ncols);
      for (int c = 0; c < ncols; c++) col[c] += (i128)qint[t] * acc[c];
    }
    if (rndb(col, ncols, Wd, U + (size_t)m * Wd)) rc = 1;
  }
  for (int i = 0; i < N && !rc; i++) {
    const int32_t *C = Cb + (size_t)i * Wd;
    for (int m = 0; m < D; m++) {
      i128 *x = X + (size_t)m * (ncols + 8);
      memset(x, 0, sizeof(i128) * ncols);
      tprod_acc(U + (size_t)m * Wd, C, L, Lf + sc - 2, x, ncols);
      if (rndb(x, ncols, Wd, CO(m, i + 1))) rc = 1;
    }
    if (i + 1 >= N) break;
    for (int e = 0; e < D * D; e++) {
      if (!snz[e]) continue;
      memset(col, 0, sizeof(i128) * ncols);
      tprod_acc(S + (size_t)e * Wd, C, L, Lf - 2, col, ncols);
      if (rndb(col, ncols, KW, K + (size_t)e * KW)) rc = 1;
    }
    const int j = i + 1;
    for (int m = 0; m < D; m++) {
      memset(col, 0, sizeof(i128) * ncols);
      for (int jj = 0; jj < D; jj++) {
        if (linI[m * D + jj]) {
          const i128 *x = X + (size_t)jj * (ncols + 8);
          for (int c = 0; c < ncols; c++) col[c] += (i128)linI[m * D + jj] * x[c];
        }
        if (snz[m * D + jj])
          tprod_acc2(U + (size_t)jj * Wd, L, K + ((size_t)m * D + jj) * KW, KW, Lf + sc - 2, col, ncols);
      }
      for (int t = 0; t < M->NT; t++) {
        if (M->teq[t] != m) continue;
        const int a = M->tj[t], b = M->tk[t];
        memset(acc, 0, sizeof(i128) * ncols);
        if (j == 2) tprod_acc(CO(a, 1), CO(b, 1), L, Lf - 2, acc, ncols);
        if (j >= 3) {
          tprod_acc(CO(a, j - 1), CO(b, 1), L, Lf - 2, acc, ncols);
          tprod_acc(CO(a, 1), CO(b, j - 1), L, Lf - 2, acc, ncols);
        }
        for (int k = 2; k <= j - 2; k++) tprod_acc(CO(a, j - k), CO(b, k), L, Lf - 2, acc, ncols);
        for (int c = 0; c < ncols; c++) col[c] += (i128)qint[t] * acc[c];
      }
      if (rndb(col, ncols, Wd, U2 + (size_t)m * Wd)) rc = 1;
    }
    memcpy(U, U2, sizeof(int32_t) * (size_t)D * Wd);
  }
#undef CO
  free(col);
  free(X);
  free(SB);
  free(S);
  free(K);
  free(Cb);
  free(U);
  free(U2);
  return rc;
}

/* ---------------------------------------------------------------------------
 * Value-exact direct recurrence (variant 3; paper_1908_09301_b200/csrc/taylor_warp.cu,
 * one warp per trajectory). The per-order recurrence of variant 0 with every
 * rounding a function of the VALUE of an exact column sum only (sd_cols), so
 * the device may skip zero digits, fold and reduce its partial sums in any
 * order and still agree bit for bit:
 *
 *   a~_0^m   = sd(state^m)                                    (same value, recoded)
 *   U_i^m    = rndb( [i==0] cst_m B^2 + sum_j tprod(lin[m][j], a~_i^j)
 *                    + sum_{t in m} q_t sum_{k=0..i} tprod(a~^a_{i-k}, a~^b_k) )
 *   a~_{i+1}^m = rndb( tprod(U_i^m, C_i, Lf+sc-2) )
 * (tprod without a T argument: T = Lf-2.) Requires small-integer bilinear
 * coefficients. The state update is the exact row sum rounded to P bits, as in
 * every variant.
 */
static int jet_wp(const model_t *M, int32_t *coef) {
  int Lf = M->Lf, L = Lf + 1, Wd = W(M), D = M->D, N = M->order;
  int ncols = Lf + 4;
  int64_t qint[64];
  for (int t = 0; t < M->NT; t++)
    if (!small_int(M->q + (size_t)t * Wd, Lf, &qint[t])) return -5;
  i128 *col = malloc(sizeof(i128) * (size_t)(ncols + 8));
  i128 *acc = malloc(sizeof(i128) * (size_t)(ncols + 8));
  int32_t *U = malloc(sizeof(int32_t) * (size_t)D * Wd);
  int rc = 0;
#define CO(m, i) (coef + ((size_t)(m) * (N + 1) + (i)) * Wd)
  for (int m = 0; m < D && !rc; m++) {
    for (int d = 0; d <= Lf; d++) acc[d] = CO(m, 0)[d];
    if (sd_cols(acc, Wd, 0, 0, Wd, CO(m, 0))) rc = 1;
  }
  for (int i = 0; i < N && !rc; i++) {
    for (int m = 0; m < D; m++) {
      memset(col, 0, sizeof(i128) * ncols);
      if (i == 0)
        for (int j = 0; j <= Lf; j++) col[2 + j] += (i128)M->cst[(size_t)m * Wd + j];
      for (int j = 0; j < D; j++) tprod_acc(M->lin + ((size_t)m * D + j) * Wd, CO(j, i), L, Lf - 2, col, ncols);
      for (int t = 0; t < M->NT; t++) {
        if (M->teq[t] != m) continue;
        memset(acc, 0, sizeof(i128) * ncols);
        for (int k = 0; k <= i; k++) tprod_acc(CO(M->tj[t], i - k), CO(M->tk[t], k), L, Lf - 2, acc, ncols);
        for (int c = 0; c < ncols; c++) col[c] += (i128)qint[t] * acc[c];
      }
      if (rndb(col, ncols, Wd, U + (size_t)m * Wd)) rc = 1;
    }
    for (int m = 0; m < D; m++) {
      memset(col, 0, sizeof(i128) * ncols);
      tprod_acc(U + (size_t)m * Wd, M->ctab + (size_t)i * Wd, L, Lf + M->sc - 2, col, ncols);
      if (rndb(col, ncols, Wd, CO(m, i + 1))) rc = 1;
    }
  }
#undef CO
  free(col);
  free(acc);
  free(U);
  return rc;
}

static int jet_any(const model_t *M, int32_t *coef) {
  return M->variant == 3 ? jet_wp(M, coef)
         : M->variant == 2 ? jet_lx(M, coef) : M->variant == 1 ? jet_mx(M, coef) : jet(M, coef);
}

/* round the canonical digit vector to `prec` significant bits, ties to even */
static int round_prec(int32_t *d, int W, int prec) {
  int tp = -1;
  for (int j = W - 1; j >= 0; j--)
    if (d[j]) { tp = j; break; }
  if (tp < 0) return 0;
  int neg = d[tp] < 0;
  i128 mag = 0;  /* not big enough in general: work digit-wise */
  (void)mag;
  int64_t m[4096 + 8];
  for (int j = 0; j < W; j++) m[j] = d[j] < 0 ? -(int64_t)d[j] : d[j];
  int tb = 0;
  while ((m[tp] >> tb) != 0) tb++;
  int nbits = RADIX_BITS * tp + tb;
  int s = nbits - prec;
  if (s <= 0) return 0;
  int sd = s / RADIX_BITS, sb = s % RADIX_BITS;
  int hp = s - 1, hd = hp / RADIX_BITS, hb = hp % RADIX_BITS;
  int half = (int)((m[hd] >> hb) & 1);
  int lsb = (int)((m[sd] >> sb) & 1);
  int sticky = (m[hd] & (((int64_t)1 << hb) - 1)) != 0;
  for (int j = 0; j < hd; j++) sticky |= m[j] != 0;
  for (int j = 0; j < sd; j++) m[j] = 0;
  m[sd] &= ~(((int64_t)1 << sb) - 1);
  if (half && (sticky || lsb)) {
    int64_t cin = (int64_t)1 << sb;
    for (int j = sd; j < W && cin; j++) {
      m[j] += cin;
      cin = m[j] >> RADIX_BITS;
      m[j] &= RADIX - 1;
    }
    if (cin) return 1;
  }
  for (int j = 0; j < W; j++) d[j] = (int32_t)(neg ? -m[j] : m[j]);
  return 0;
}

/* exact sum of the rows: state[m] = sum_i coef[m][i] */
static int sum_rows(const model_t *M, const int32_t *coef, int32_t *state, int prec) {
  int Lf = M->Lf, Wd = W(M), N = M->order;
  i128 col[4096 + 8];
  int rc = 0;
  for (int m = 0; m < M->D; m++) {
    /* reuse round_cols with two zero guard columns in front */
    memset(col, 0, sizeof(i128) * (Wd + 3));
    for (int i = 0; i <= N; i++)
      for (int j = 0; j <= Lf; j++) col[2 + j] += (i128)coef[((size_t)m * (N + 1) + i) * Wd + j];
    if (round_cols_canon(col, Wd + 3, Lf, state + (size_t)m * Wd)) rc = 1;
    if (round_prec(state + (size_t)m * Wd, Wd, prec)) rc = 1;
  }
  return rc;
}

int fix_compute_jet_v(int variant, int D, int NT, const int32_t *teq, const int32_t *tj, const int32_t *tk, int Lf,
                    int sc, int order, const int32_t *cst, const int32_t *lin, const int32_t *q,
                    const int32_t *ctab, const int32_t *state, int32_t *coef_out) {
  model_t M;
  int rc = build(&M, D, NT, teq, tj, tk);
  if (rc) return rc;
  if (Lf + 4 > 4096) return -4;
  M.Lf = Lf;
  M.sc = sc;
  M.order = order;
  M.cst = cst;
  M.lin = lin;
  M.q = q;
  M.ctab = ctab;
  M.variant = variant;
  int Wd = Lf + 1;
  for (int m = 0; m < D; m++)
    memcpy(coef_out + (size_t)m * (order + 1) * Wd, state + (size_t)m * Wd, sizeof(int32_t) * Wd);
  return jet_any(&M, coef_out);
}

/* records: step start, every multiple of stride, and n_steps; returns #records or <0 */
int fix_integrate_v(int variant, int D, int NT, const int32_t *teq, const int32_t *tj, const int32_t *tk, int Lf,
                  int sc, int order, int prec, const int32_t *cst, const int32_t *lin, const int32_t *q,
                  const int32_t *ctab, const int32_t *state0, int n_steps, int start_step,
                  int stride, int max_rec, int32_t *rec_step, int32_t *rec_state) {
  model_t M;
  int rc = build(&M, D, NT, teq, tj, tk);
  if (rc) return rc;
  if (Lf + 4 > 4096) return -4;
  M.Lf = Lf;
  M.sc = sc;
  M.order = order;
  M.cst = cst;
  M.lin = lin;
  M.q = q;
  M.ctab = ctab;
  M.variant = variant;
  int Wd = Lf + 1;
  int32_t *coef = malloc(sizeof(int32_t) * (size_t)D * (order + 1) * Wd);
  int32_t *state = malloc(sizeof(int32_t) * (size_t)D * Wd);
  memcpy(state, state0, sizeof(int32_t) * (size_t)D * Wd);
  int nrec = 0;
  rc = 0;
  if (max_rec < 1) { rc = -2; goto out; }
  rec_step[nrec] = start_step;
  memcpy(rec_state, state, sizeof(int32_t) * (size_t)D * Wd);
  nrec++;
  for (int n = start_step + 1; n <= n_steps; n++) {
    for (int m = 0; m < D; m++)
      memcpy(coef + (size_t)m * (order + 1) * Wd, state + (size_t)m * Wd, sizeof(int32_t) * Wd);
    if (jet_any(&M, coef) || sum_rows(&M, coef, state, prec)) { rc = -1; goto out; }
    if (n % stride == 0 || n == n_steps) {
      if (nrec >= max_rec) { rc = -2; goto out; }
      rec_step[nrec] = n;
      memcpy(rec_state + (size_t)nrec * D * Wd, state, sizeof(int32_t) * (size_t)D * Wd);
      nrec++;
    }
  }
out:
  free(coef);
  free(state);
  return rc < 0 ? rc : nrec;
}

int fix_compute_jet(int D, int NT, const int32_t *teq, const int32_t *tj, const int32_t *tk, int Lf, int sc,
                    int order, const int32_t *cst, const int32_t *lin, const int32_t *q, const int32_t *ctab,
                    const int32_t *state, int32_t *coef_out) {
  return fix_compute_jet_v(0, D, NT, teq, tj, tk, Lf, sc, order, cst, lin, q, ctab, state, coef_out);
}

int fix_integrate(int D, int NT, const int32_t *teq, const int32_t *tj, const int32_t *tk, int Lf, int sc,
                  int order, int prec, const int32_t *cst, const int32_t *lin, const int32_t *q,
                  const int32_t *ctab, const int32_t *state0, int n_steps, int start_step, int stride,
                  int max_rec, int32_t *rec_step, int32_t *rec_state) {
  return fix_integrate_v(0, D, NT, teq, tj, tk, Lf, sc, order, prec, cst, lin, q, ctab, state0, n_steps,
                         start_step, stride, max_rec, rec_step, rec_state);
}
