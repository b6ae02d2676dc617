/*
 * Minimal declarations of the MPFR 4.x / GMP 6.x ABI used by the oracle.
 *
 * TEST INFRASTRUCTURE ONLY. The image ships libmpfr.so.6 (MPFR 4.2.1) and
 * libgmp.so.10 (GMP 6.3.0) but not their headers; the reference package's
 * arithmetic backend is gmpy2 -> MPFR, so linking the same library gives
 * the oracle the reference's exact rounding behaviour. Only the handful of
 * entry points the oracle calls are declared, with the ABI of the default
 * x86-64 build (mpfr_prec_t = long, mpfr_exp_t = long, 64-bit limbs).
 */
#pragma once
#include <stddef.h>
#include <stdint.h>

typedef unsigned long mp_limb_t;
typedef long mpfr_prec_t;
typedef int mpfr_sign_t;
typedef long mpfr_exp_t;

typedef struct {
  mpfr_prec_t _mpfr_prec;
  mpfr_sign_t _mpfr_sign;
  mpfr_exp_t _mpfr_exp;
  mp_limb_t *_mpfr_d;
} __mpfr_struct;
typedef __mpfr_struct mpfr_t[1];
typedef __mpfr_struct *mpfr_ptr;
typedef const __mpfr_struct *mpfr_srcptr;

typedef enum {
  MPFR_RNDN = 0,
  MPFR_RNDZ,
  MPFR_RNDU,
  MPFR_RNDD,
  MPFR_RNDA,
  MPFR_RNDF
} mpfr_rnd_t;

typedef struct {
  int _mp_alloc;
  int _mp_size;
  mp_limb_t *_mp_d;
} __mpz_struct;
typedef __mpz_struct mpz_t[1];

#ifdef __cplusplus
extern "C" {
#endif
void mpfr_init2(mpfr_ptr, mpfr_prec_t);
void mpfr_clear(mpfr_ptr);
int mpfr_set4(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t, int);
int mpfr_set_ui(mpfr_ptr, unsigned long, mpfr_rnd_t);
int mpfr_mul(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_add(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_sub(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_div(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_div_ui(mpfr_ptr, mpfr_srcptr, unsigned long, mpfr_rnd_t);
int mpfr_neg(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_zero_p(mpfr_srcptr);
int mpfr_signbit(mpfr_srcptr);
int mpfr_set_z_2exp(mpfr_ptr, const __mpz_struct *, mpfr_exp_t, mpfr_rnd_t);
mpfr_exp_t mpfr_get_z_2exp(__mpz_struct *, mpfr_srcptr);
const char *mpfr_get_version(void);

void __gmpz_init(__mpz_struct *);
void __gmpz_clear(__mpz_struct *);
void __gmpz_import(__mpz_struct *, size_t, int, size_t, int, size_t, const void *);
void *__gmpz_export(void *, size_t *, int, size_t, int, size_t, const __mpz_struct *);
void __gmpz_neg(__mpz_struct *, const __mpz_struct *);
#ifdef __cplusplus
}
#endif

#define mpfr_set(a, b, r) mpfr_set4((a), (b), (r), (b)->_mpfr_sign)
