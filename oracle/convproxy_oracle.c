/*
 * convproxy_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker).
 *
 * A plain-C restatement of the convproxy column physics, written from the
 * reference's documented formulas and checked line by line against
 *   /root/reference/proj/src/core/physics.cpp   (kernels, generator)
 *   /root/reference/proj/src/core/physics.hpp   (contracts, constants)
 *   /root/reference/proj/src/core/prng.hpp      (counter-based splitmix64)
 * Every function cites the reference lines it restates.  Compile with
 * -ffp-contract=off (as the reference's CMakeLists.txt:15 does) so that each
 * operation rounds exactly as the reference's does; exp/sin come from the
 * same libm, so on one host this oracle is bit-identical to the reference
 * (pinned by tests/test_oracle.py against oracle/_ref and tests/golden/).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this file's library; the CUDA product path never calls it.
 */
#include "convproxy_oracle.h"

#include <math.h>
#include <stddef.h>

#if defined(__FP_FAST_FMA) && !defined(ORACLE_ALLOW_CONTRACT)
/* Contraction is a compile flag, not a macro we can see; this guard only
 * documents intent.  The Makefile passes -ffp-contract=off. */
#endif

void orc_default_options(orc_options* o) {
  /* physics.hpp:68-73 */
  o->variant = ORC_EXACT;
  o->activity_threshold = 0.5;
  o->newton_tol = 1e-12;
  o->newton_max_iter = 100;
}

/* prng.hpp:27-32 */
static uint64_t splitmix_fin(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* prng.hpp:37-41 */
uint64_t orc_rng_u64(uint64_t seed, uint64_t stream, uint64_t counter) {
  const uint64_t gamma = 0x9e3779b97f4a7c15ULL; /* prng.hpp:25 */
  const uint64_t keyed = splitmix_fin(seed + gamma * (stream + 1));
  return splitmix_fin(keyed + gamma * (counter + 1));
}

/* prng.hpp:44-47 */
double orc_rng_u01(uint64_t seed, uint64_t stream, uint64_t counter) {
  return (double)(orc_rng_u64(seed, stream, counter) >> 11) * 0x1.0p-53;
}

/* physics.cpp:29-32 (Cody-Waite split of ln2) */
static const double kLn2Hi = 6.93147180369123816490e-01;
static const double kLn2Lo = 1.90821492927058770002e-10;
static const double kInvLn2 = 1.44269504088896338700e+00;

/* physics.cpp:40-60: k = nearbyint(x/ln2), r = (x - k*hi) - k*lo, degree-12
 * Horner in r, scaled by ldexp.  The domain assert (|x| <= 64) is compiled
 * out under NDEBUG in the reference and is not restated. */
double orc_approx_exp(double x) {
  const double kd = nearbyint(x * kInvLn2);
  const int k = (int)kd;
  const double r = (x - kd * kLn2Hi) - kd * kLn2Lo;
  double p = 1.0 / 479001600.0;
  p = p * r + 1.0 / 39916800.0;
  p = p * r + 1.0 / 3628800.0;
  p = p * r + 1.0 / 362880.0;
  p = p * r + 1.0 / 40320.0;
  p = p * r + 1.0 / 5040.0;
  p = p * r + 1.0 / 720.0;
  p = p * r + 1.0 / 120.0;
  p = p * r + 1.0 / 24.0;
  p = p * r + 1.0 / 6.0;
  p = p * r + 0.5;
  p = p * r + 1.0;
  p = p * r + 1.0;
  return ldexp(p, k);
}

/* The libm exp the reference calls for Exact/StrengthReduced (physics.cpp:35;
 * glibc 2.39, not vendored, reached through <cmath>), restated
 * so the device can evaluate it bit for bit (colmath.cuh exp_gl).  glibc's
 * published algorithm (sysdeps/ieee754/dbl-64/e_exp.c, table-driven, N = 128,
 * degree-5 polynomial; its FMA build on x86-64 contracts the main path's
 * multiply-adds):
 *   k = round(x 128/ln2), r = x - k ln2/128 (two-part constant),
 *   exp(x) = 2^(k/128) (1 + tail_j + r + r^2 (C2 + r C3) + r^4 (C4 + r C5)),
 * with the scaled special case for |x| in [512, 1024) (contracted for k > 0,
 * uncontracted in the subnormal branch -- as measured against the libm) and
 * 1 + x for |x| < 2^-54.  The table comes from tools/gen_exp_table.py (own
 * computation); tests/test_oracle.py pins this restatement against the
 * running libm over millions of arguments. */
#include <string.h>
#include "../paper_1711_00289_b200/csrc/exp_gl_table.h"
static const uint64_t kExpGlTab[256] = {CVG_EXP_GL_TABLE};
static uint64_t dbits(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
static double bitsd(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }

static double exp_gl_special(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000u) == 0) {      /* k > 0: scale's exponent overflowed */
    const double scale = bitsd(sbits - (1009ull << 52));
    return 0x1p1009 * fma(scale, tmp, scale);
  }
  const double scale = bitsd(sbits + (1022ull << 52));  /* k < 0: subnormal range */
  const double st = scale * tmp;
  double y = scale + st;
  if (y < 1.0) {
    double lo = (scale - y) + st;
    const double hi = 1.0 + y;
    lo = ((1.0 - hi) + y) + lo;
    y = (hi + lo) - 1.0;
    if (y == 0.0) y = 0.0;
  }
  return 0x1p-1022 * y;
}

double orc_exp_gl(double x) {
  uint32_t abstop = (uint32_t)(dbits(x) >> 52) & 0x7ff;
  if (abstop - 0x3c9u >= 0x408u - 0x3c9u) {          /* |x| < 2^-54 or >= 512 */
    if (abstop - 0x3c9u >= 0x80000000u) return 1.0 + x;
    if (abstop >= 0x409u) {                           /* |x| >= 1024, inf, nan */
      if (dbits(x) == dbits(-INFINITY)) return 0.0;
      if (abstop >= 0x7ffu) return 1.0 + x;
      return (dbits(x) >> 63) ? 0.0 : INFINITY;
    }
    abstop = 0;
  }
  double kd = fma(0x1.71547652b82fep7, x, 0x1.8p52);
  const uint64_t ki = dbits(kd);
  kd -= 0x1.8p52;
  const double r = fma(kd, -0x1.cf79abc9e3b3ap-47, fma(kd, -0x1.62e42fefa0000p-8, x));
  const uint64_t idx = 2 * (ki % 128);
  const double tail = bitsd(kExpGlTab[idx]);
  const uint64_t sbits = kExpGlTab[idx + 1] + (ki << 45);
  const double r2 = r * r;
  const double tmp = fma(r2 * r2, fma(r, 0x1.1111167a4d017p-7, 0x1.55555cf172b91p-5),
                         fma(r2, fma(r, 0x1.555555555543cp-3, 0x1.ffffffffffdbdp-2), tail + r));
  if (abstop == 0) return exp_gl_special(tmp, sbits, ki);
  const double scale = bitsd(sbits);
  return fma(scale, tmp, scale);
}

/* Vector forms for the pinning test: the restatement and the running libm. */
void orc_exp_gl_vec(long long n, const double* x, double* out) {
  for (long long i = 0; i < n; ++i) out[i] = orc_exp_gl(x[i]);
}
void orc_libm_exp_vec(long long n, const double* x, double* out) {
  for (long long i = 0; i < n; ++i) out[i] = exp(x[i]);
}

/* physics.cpp:34-36 */
static double exp_eval(double x, int variant) {
  return variant == ORC_APPROX_TRANSCENDENTAL ? orc_approx_exp(x) : exp(x);
}

static double margin_of(double resid, double tol) {
  return fabs(fabs(resid) - tol) / tol;
}

/* physics.cpp:64-87.  Up to max_iter+1 convergence tests; a test passing
 * after `it` updates returns it.  Tracks the Newton-margin classifier. */
static int ientropy_impl(double y, double guess, const orc_options* o,
                         double* root, int* iters, double* min_margin) {
  if (!isfinite(y) || !isfinite(guess)) return ORC_FAIL_INPUT;
  double t = guess;
  double e = exp_eval(0.05 * t, o->variant);
  double resid = e + 0.01 * t - y;
  for (int it = 0; it <= o->newton_max_iter; ++it) {
    if (min_margin) {
      const double m = margin_of(resid, o->newton_tol);
      if (m < *min_margin) *min_margin = m;
    }
    if (fabs(resid) <= o->newton_tol) {
      *root = t;
      *iters = it;
      return ORC_OK;
    }
    const double deriv = 0.05 * e + 0.01;
    t -= resid / deriv;
    if (!isfinite(t)) return ORC_FAIL_DIVERGED;
    e = exp_eval(0.05 * t, o->variant);
    resid = e + 0.01 * t - y;
  }
  return ORC_FAIL_NOCONV;
}

int orc_ientropy_solve(double y, double guess, const orc_options* o,
                       double* root, int* iterations, double* min_margin) {
  double r = 0.0;
  int it = 0;
  if (min_margin) *min_margin = INFINITY;
  const int st = ientropy_impl(y, guess, o, &r, &it, min_margin);
  if (st == ORC_OK) {
    *root = r;
    *iterations = it;
  }
  return st;
}

/* physics.hpp:94-96 */
static double div_by_square(double num, double den, int reduced) {
  return reduced ? num / (den * den) : num / den / den;
}

/* std::max(0.0, x) returns 0.0 unless 0.0 < x (so NaN -> 0.0). */
static double max0(double x) { return (0.0 < x) ? x : 0.0; }

/* physics.cpp:106-166 for one column; column c of the SoA block. */
static int deep_one(long long c, int L, long long ld, const double* s,
                    const double* T, const double* q, const orc_options* o,
                    double* tend_T, double* tend_q, double* precip,
                    long long* work, unsigned char* exited, double* margin) {
  const double sc = s[c];
  if (margin) margin[c] = INFINITY;
  if (!isfinite(sc)) return ORC_FAIL_ACTIVITY;           /* :108-110 */
  if (sc <= o->activity_threshold) {                     /* :111-113 */
    for (int k = 0; k < L; ++k) {
      tend_T[k * ld + c] = 0.0;
      tend_q[k * ld + c] = 0.0;
    }
    precip[c] = 0.0;
    work[c] = 0;
    exited[c] = 1;
    return ORC_OK;
  }
  const int reduced = o->variant == ORC_STRENGTH_REDUCED;
  const double guess = 24.0 + 160.0 * sc;                /* :121 */
  const double rho = 1.0 + 0.05 * sc;                    /* :127 / :146 */
  long long w = 0;
  double mm = INFINITY;
  /* entrainment pass, :129-135 / :145-153 */
  for (int k = 0; k < L; ++k) {
    const double Tk = T[k * ld + c], qk = q[k * ld + c];
    const double m = div_by_square(qk, rho, reduced);
    const double ye = 1.0 + 1.0e-3 * Tk + 0.1 * m;
    double re = 0.0;
    int it = 0;
    const int st = ientropy_impl(ye, guess, o, &re, &it, &mm);
    if (st != ORC_OK) return st;
    w += it;
    tend_T[k * ld + c] =
        0.02 * (250.0 + 2.0 * re - Tk) + 0.3 * sin(6.0 * Tk + 50.0 * qk);
  }
  /* precipitation pass, :136-143 / :154-162; precip summed in k order */
  double pr = 0.0;
  for (int k = 0; k < L; ++k) {
    const double Tk = T[k * ld + c], qk = q[k * ld + c];
    const double m = div_by_square(qk, rho, reduced);
    const double yp = 1.0 + 8.0e-4 * Tk + 0.05 * m + 0.1 * sc;
    double rp = 0.0;
    int it = 0;
    const int st = ientropy_impl(yp, guess, o, &rp, &it, &mm);
    if (st != ORC_OK) return st;
    w += it;
    tend_q[k * ld + c] = 0.05 * (0.01 + 0.002 * sin(3.0 * rp) - qk);
    pr += qk * max0(rp - 4.5);
  }
  precip[c] = pr;
  work[c] = w;
  exited[c] = 0;
  if (margin) margin[c] = mm;
  return ORC_OK;
}

/* physics.cpp:227-235 */
int orc_deep_convection(long long n, int L, long long ld, long long first_col,
                        const double* s, const double* T, const double* q,
                        const orc_options* o, double* tend_T, double* tend_q,
                        double* precip, long long* work, unsigned char* exited,
                        double* newton_margin, long long* fail_col) {
  for (long long c = 0; c < n; ++c) {
    const int st = deep_one(c, L, ld, s, T, q, o, tend_T, tend_q, precip, work,
                            exited, newton_margin);
    if (st != ORC_OK) {
      if (fail_col) *fail_col = first_col + c;
      return st;
    }
  }
  return ORC_OK;
}

/* physics.cpp:168-225 */
static const double kW1[4] = {0.8, 1.1, 0.9, 1.2};     /* :174 */
static const double kW2[4] = {30.0, 20.0, 40.0, 25.0}; /* :175 */
static const double kW3[4] = {0.5, 0.3, 0.4, 0.2};     /* :176 */
static const double kTheta[4] = {0.15, 0.30, 0.45, 0.60}; /* physics.hpp:149 */

static int shallow_one(long long c, int L, long long ld, const double* s,
                       const double* T, const double* q, const orc_options* o,
                       double* tend_T, double* tend_q, double* precip,
                       long long* work, unsigned char* exited,
                       double* margin) {
  const double sc = s[c];
  if (margin) margin[c] = INFINITY;
  if (!isfinite(sc)) return ORC_FAIL_ACTIVITY;          /* :171-173 */
  const int reduced = o->variant == ORC_STRENGTH_REDUCED;
  const double rho = 1.0 + 0.05 * sc;
  double acc = 0.0;
  long long w = 0;
  double mm = INFINITY;
  for (int j = 0; j < 4; ++j) {                          /* :182 */
    double phase_sum = 0.0;
    for (int k = 0; k < L; ++k) {
      const double Tk = T[k * ld + c], qk = q[k * ld + c];
      double term = 1.0e-3 * kW1[j] * Tk + kW2[j] * div_by_square(qk, rho, reduced);
      if (j == 1) term += 0.02 * exp_eval(-50.0 * qk, o->variant);
      phase_sum += term;
    }
    acc += phase_sum / (double)L + kW3[j] * sc;          /* :205 */
    w += L;                                              /* :206 */
    const double lhs = sc * (1.0 + 0.05 * sin(3.0 * acc));
    const double mg = fabs(lhs - kTheta[j]) / kTheta[j];
    if (mg < mm) mm = mg;
    if (lhs < kTheta[j]) {                               /* :207-211 */
      for (int k = 0; k < L; ++k) {
        tend_T[k * ld + c] = 0.0;
        tend_q[k * ld + c] = 0.0;
      }
      precip[c] = 0.0;
      work[c] = w;
      exited[c] = 1;
      if (margin) margin[c] = mm;
      return ORC_OK;
    }
  }
  const double sa = sin(acc);                            /* :214-224 */
  for (int k = 0; k < L; ++k) {
    const double Tk = T[k * ld + c], qk = q[k * ld + c];
    tend_T[k * ld + c] = 0.005 * (256.0 + 2.0 * sa - Tk);
    tend_q[k * ld + c] = 0.02 * (0.012 - qk);
  }
  precip[c] = (sc - 0.5) * max0(sa + 0.5);
  work[c] = w;
  exited[c] = 0;
  if (margin) margin[c] = mm;
  return ORC_OK;
}

/* physics.cpp:237-245 */
int orc_shallow_convection(long long n, int L, long long ld,
                           long long first_col, const double* s,
                           const double* T, const double* q,
                           const orc_options* o, double* tend_T,
                           double* tend_q, double* precip, long long* work,
                           unsigned char* exited, double* pred_margin,
                           long long* fail_col) {
  for (long long c = 0; c < n; ++c) {
    const int st = shallow_one(c, L, ld, s, T, q, o, tend_T, tend_q, precip,
                               work, exited, pred_margin);
    if (st != ORC_OK) {
      if (fail_col) *fail_col = first_col + c;
      return st;
    }
  }
  return ORC_OK;
}

/* physics.cpp:247-277 (make_column / make_grid), level-major output. */
void orc_make_grid(long long n, int L, double tropics_band, uint64_t seed,
                   double* s, double* T, double* q) {
  const long long band = llround(tropics_band * (double)n);
  const long long lo = (n - band) / 2;
  for (long long c = 0; c < n; ++c) {
    const int tropical = c >= lo && c < lo + band;
    const double us = orc_rng_u01(seed, 0, (uint64_t)c);
    s[c] = tropical ? 0.5 + 0.5 * us : 0.5 * us;
    for (int k = 0; k < L; ++k) {
      const uint64_t ctr = (uint64_t)c * (uint64_t)L + (uint64_t)k;
      T[(long long)k * n + c] = 250.0 + 60.0 * orc_rng_u01(seed, 1, ctr);
      q[(long long)k * n + c] = 0.022 * orc_rng_u01(seed, 2, ctr);
    }
  }
}
