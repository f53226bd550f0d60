/* Declaration-only shim for the 11 MPFR 4.2 entry points used by the
 * reference's oracle.cpp (proj/src/oracle.cpp:105-127).  The container ships
 * libmpfr.so.6 / libgmp.so.10 but no headers, so the reference's
 * find_library(mpfr REQUIRED) (proj/src/CMakeLists.txt:25-26) cannot be used;
 * this header lets g++ compile oracle.cpp unchanged and link against the
 * versioned shared objects.  Test infrastructure only. */
#ifndef JT_MPFR_SHIM_H
#define JT_MPFR_SHIM_H
#ifdef __cplusplus
extern "C" {
#endif
typedef long mpfr_prec_t;
typedef int mpfr_sign_t;
typedef long mpfr_exp_t;
typedef unsigned long mp_limb_t;
typedef struct {
  mpfr_prec_t _mpfr_prec;
  mpfr_sign_t _mpfr_sign;
  mpfr_exp_t _mpfr_exp;
  mp_limb_t *_mpfr_d;
} __mpfr_struct;
typedef __mpfr_struct mpfr_t[1];
typedef __mpfr_struct *mpfr_ptr;
typedef const __mpfr_struct *mpfr_srcptr;
typedef enum { MPFR_RNDN = 0, MPFR_RNDZ, MPFR_RNDU, MPFR_RNDD, MPFR_RNDA } mpfr_rnd_t;
mpfr_exp_t mpfr_get_emin(void);
mpfr_exp_t mpfr_get_emax(void);
int mpfr_set_emin(mpfr_exp_t);
int mpfr_set_emax(mpfr_exp_t);
void mpfr_init2(mpfr_ptr, mpfr_prec_t);
void mpfr_clear(mpfr_ptr);
int mpfr_strtofr(mpfr_ptr, const char *, char **, int, mpfr_rnd_t);
int mpfr_check_range(mpfr_ptr, int, mpfr_rnd_t);
int mpfr_subnormalize(mpfr_ptr, int, mpfr_rnd_t);
double mpfr_get_d(mpfr_srcptr, mpfr_rnd_t);
int mpfr_inf_p(mpfr_srcptr);
#ifdef __cplusplus
}
#endif
#endif
