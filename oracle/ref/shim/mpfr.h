/* Declaration-only MPFR header for compiling the reference's kernel.cpp
 * against the runtime libmpfr.so.6 shipped in this image (its development
 * header is not installed). Only the entry points kernel.cpp:131-222 use are
 * declared; layouts follow the MPFR 4 ABI (long precision/exponent). */
#pragma once
#ifdef __cplusplus
extern "C" {
#endif
typedef long mpfr_prec_t;
typedef int mpfr_sign_t;
typedef long mpfr_exp_t;
typedef struct {
    mpfr_prec_t _mpfr_prec;
    mpfr_sign_t _mpfr_sign;
    mpfr_exp_t _mpfr_exp;
    unsigned long* _mpfr_d;
} __mpfr_struct;
typedef __mpfr_struct mpfr_t[1];
typedef __mpfr_struct* mpfr_ptr;
typedef const __mpfr_struct* mpfr_srcptr;
typedef enum { MPFR_RNDN = 0, MPFR_RNDZ, MPFR_RNDU, MPFR_RNDD, MPFR_RNDA } mpfr_rnd_t;

void mpfr_inits2(mpfr_prec_t, mpfr_ptr, ...);
void mpfr_clears(mpfr_ptr, ...);
int mpfr_set_d(mpfr_ptr, double, mpfr_rnd_t);
int mpfr_set_ui(mpfr_ptr, unsigned long, mpfr_rnd_t);
void mpfr_set_inf(mpfr_ptr, int);
int mpfr_set4(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t, int);
int mpfr_sqr(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_add(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_sub(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_mul(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_div(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_neg(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_mul_d(mpfr_ptr, mpfr_srcptr, double, mpfr_rnd_t);
int mpfr_add_ui(mpfr_ptr, mpfr_srcptr, unsigned long, mpfr_rnd_t);
int mpfr_cmp3(mpfr_srcptr, mpfr_srcptr, int);
double mpfr_get_d(mpfr_srcptr, mpfr_rnd_t);
#ifdef __cplusplus
}
#endif
#define MPFR_SIGN(x) ((x)->_mpfr_sign)
#define mpfr_set(a, b, r) mpfr_set4(a, b, r, MPFR_SIGN(b))
#define mpfr_cmp(b, c) mpfr_cmp3(b, c, 1)
