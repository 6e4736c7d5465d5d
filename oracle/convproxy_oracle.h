/*
 * convproxy_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's column-physics hot path
 * (/root/reference/proj/src/core/physics.cpp, prng.hpp) used as the parity
 * checker for the CUDA path.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load this library.  The product library
 * (libconvgpu.so) never links or calls it.
 *
 * Data layout matches the product C-ABI: level-major structure of arrays,
 * field[k * ld + c] for level k of column c, ld >= n.
 */
#ifndef CONVPROXY_ORACLE_H_
#define CONVPROXY_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors convproxy::Variant (physics.hpp:62-66). */
enum { ORC_EXACT = 0, ORC_STRENGTH_REDUCED = 1, ORC_APPROX_TRANSCENDENTAL = 2 };

/* Failure kinds, in the order the reference can raise them for one column. */
enum {
  ORC_OK = 0,
  ORC_FAIL_ACTIVITY = 1,    /* non-finite s            physics.cpp:108-110, :171-173 */
  ORC_FAIL_INPUT = 2,       /* non-finite y or guess   physics.cpp:66-68 */
  ORC_FAIL_DIVERGED = 3,    /* non-finite iterate      physics.cpp:78-80 */
  ORC_FAIL_NOCONV = 4       /* max_iter exceeded       physics.cpp:84-86 */
};

/* Mirrors convproxy::KernelOptions (physics.hpp:68-73). */
typedef struct orc_options {
  int variant;
  double activity_threshold;
  double newton_tol;
  int newton_max_iter;
} orc_options;

void orc_default_options(orc_options* o);

/* splitmix64 counter-based generator, prng.hpp:23-47. */
uint64_t orc_rng_u64(uint64_t seed, uint64_t stream, uint64_t counter);
double orc_rng_u01(uint64_t seed, uint64_t stream, uint64_t counter);

/* physics.cpp:40-60 */
double orc_approx_exp(double x);

/* glibc 2.39 exp restated (the libm exp of physics.cpp:35); vector forms of
 * it and of the running libm exp, for the pinning test. */
double orc_exp_gl(double x);
void orc_exp_gl_vec(long long n, const double* x, double* out);
void orc_libm_exp_vec(long long n, const double* x, double* out);

/* physics.cpp:64-87, :101-104.  Returns ORC_OK or a failure kind.
 * min_margin (nullable) receives min over convergence tests of
 * | |resid| - tol | / tol (the Newton-margin classifier). */
int orc_ientropy_solve(double y, double guess, const orc_options* o,
                       double* root, int* iterations, double* min_margin);

/* Serial chunk drivers, physics.cpp:227-245 over physics.cpp:106-166 and
 * :168-225.  Returns ORC_OK, or the failure kind of the first (lowest)
 * failing column with its id (first_col + c) in *fail_col.
 * Diagnostics (nullable): newton_margin[c] (deep) and pred_margin[c]
 * (shallow: min over executed predicates of |lhs - theta_j| / theta_j);
 * +inf when no test was evaluated. */
int orc_deep_convection(long long n, int L, long long ld, long long first_col,
                        const double* s, const double* T, const double* q,
                        const orc_options* o, double* tend_T, double* tend_q,
                        double* precip, long long* work, unsigned char* exited,
                        double* newton_margin, long long* fail_col);
int orc_shallow_convection(long long n, int L, long long ld,
                           long long first_col, const double* s,
                           const double* T, const double* q,
                           const orc_options* o, double* tend_T,
                           double* tend_q, double* precip, long long* work,
                           unsigned char* exited, double* pred_margin,
                           long long* fail_col);

/* Reference grid generator, physics.cpp:247-277, level-major output. */
void orc_make_grid(long long n, int L, double tropics_band, uint64_t seed,
                   double* s, double* T, double* q);

#ifdef __cplusplus
}
#endif
#endif
