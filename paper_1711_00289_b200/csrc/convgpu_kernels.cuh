// convgpu_kernels.cuh -- sm_100a kernels of the convection column path.
//
//   trigger_compact_kernel  deep trigger s > thr (physics.cpp:108-113) with
//                           warp-ballot / block-scan stream compaction into a
//                           dense list of triggered columns (replaces the
//                           reference's dynamic scheduling, sched.cpp:166-173)
//   deep_kernel             deep plume (physics.cpp:106-166) over the
//                           compacted list: one lane per (column, level), each
//                           lane runs its level's entrainment then
//                           precipitation Newton solve (physics.cpp:64-87);
//                           persistent blocks pull tiles of columns from an
//                           atomic cursor; ordered precip sum per column
//   shallow_kernel          shallow scheme (physics.cpp:168-225), one thread
//                           per column, streaming level-major rows, fused with
//                           the zero-fill of untriggered deep columns
//                           (physics.cpp:89-97, :111-113)
//   ientropy_kernel         batched ientropy_solve (physics.cpp:101-104)
//   approx_exp_kernel       approx_exp (physics.cpp:40-60)
//
// Layout: level-major SoA, field[k * ld + c].  Every IEEE operation of the
// reference is one uncontracted, correctly rounded device operation (see
// colmath.cuh); outputs therefore match the reference bit for bit except
// where libm exp/sin enter (Exact/StrengthReduced variants).
#pragma once
#include <cstdint>

#include "colmath.cuh"

namespace cvg {

enum : int { kVarExact = 0, kVarReduced = 1, kVarApprox = 2 };
enum : int { kFailNone = 0, kFailActivity = 1, kFailInput = 2, kFailDiverged = 3, kFailNoConv = 4 };

// Failure key: lowest column first, then the solve order the serial
// reference would have met (entrainment k, then precipitation k), then kind.
__device__ __forceinline__ void raise_failure(unsigned long long* err, long long col, int order,
                                              int kind) {
  atomicMin(err, ((unsigned long long)col << 16) | ((unsigned long long)order << 3) |
                     (unsigned long long)kind);
}

__device__ __forceinline__ double max0(double x) { return (0.0 < x) ? x : 0.0; }

// ---------------------------------------------------------------------------
// Trigger + stream compaction.  Each 1024-thread block owns a tile of 4096
// consecutive columns (4 per thread, coalesced); triggered columns of a tile
// are written contiguously and in column order (warp ballot + block scan),
// and one atomicAdd per block reserves the tile's slice of the list.
constexpr int kTrigThreads = 1024;
constexpr int kTrigPerThread = 4;
constexpr int kTrigTile = kTrigThreads * kTrigPerThread;

__global__ void __launch_bounds__(kTrigThreads)
trigger_compact_kernel(const double* __restrict__ s, long long n, double thr,
                       int* __restrict__ idx, int* __restrict__ count,
                       unsigned long long* __restrict__ err_deep) {
  __shared__ int s_cnt[kTrigPerThread * 32];
  __shared__ int s_base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long tile0 = (long long)blockIdx.x * kTrigTile;
  unsigned ballots[kTrigPerThread];
#pragma unroll
  for (int i = 0; i < kTrigPerThread; ++i) {
    const long long c = tile0 + (long long)i * kTrigThreads + threadIdx.x;
    bool f = false;
    if (c < n) {
      const double sc = s[c];
      if (!is_finite(sc)) raise_failure(err_deep, c, 0, kFailActivity);
      f = sc > thr;
    }
    ballots[i] = __ballot_sync(0xffffffffu, f);
    if (lane == 0) s_cnt[i * 32 + warp] = __popc(ballots[i]);
  }
  __syncthreads();
  if (warp == 0) {
    // exclusive scan of the 128 (i, warp) counts, in column order
    int v[kTrigPerThread];
    int tot = 0;
#pragma unroll
    for (int i = 0; i < kTrigPerThread; ++i) { v[i] = s_cnt[lane * kTrigPerThread + i]; tot += v[i]; }
    int incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    int run = incl - tot;
#pragma unroll
    for (int i = 0; i < kTrigPerThread; ++i) { const int x = v[i]; s_cnt[lane * kTrigPerThread + i] = run; run += x; }
    if (lane == 31) s_base = incl > 0 ? atomicAdd(count, incl) : 0;
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < kTrigPerThread; ++i) {
    if (ballots[i] & (1u << lane)) {
      const long long c = tile0 + (long long)i * kTrigThreads + threadIdx.x;
      idx[s_base + s_cnt[i * 32 + warp] + __popc(ballots[i] & lt)] = (int)c;
    }
  }
}

// ---------------------------------------------------------------------------
// Deep plume.
struct DeepArgs {
  const double* s;
  const double* T;
  const double* q;
  long long ld_in;
  double* tend_T;
  double* tend_q;
  double* precip;
  long long* work;
  uint8_t* exited;
  long long ld_out;
  const int* idx;         // compacted triggered columns
  const int* count;       // number of triggered columns (device)
  int* tile_cursor;       // persistent-block work cursor (zeroed per call)
  unsigned long long* err;
  const double2* exp_tab; // 2^(j/512) double-double table (global)
  long long first_col;
  double thr, tol;
  int maxit;
  int L;                  // levels
  int cpb;                // columns per tile
  bool fast_div_ok;       // newton_tol >= 2^-500
};

template <int VAR>
__device__ __forceinline__ double deep_exp(double x, const double2* tab, bool& fast) {
  if (VAR == kVarApprox) {
    fast = false;
    return approx_exp_ref(x);
  }
  fast = exp_fast_ok(x);
  return fast ? exp_tang(x, tab) : exp(x);
}

// Inverse-entropy Newton iteration for one (y, guess) solve, restating
// physics.cpp:64-87: up to max_iter+1 convergence tests, an update after
// each failed test, non-finite iterates rejected.  The two solves of a lane
// run as one flattened loop so a lane that converges its entrainment solve
// moves straight on to its precipitation solve without waiting for its
// warp.  Returns false on failure (raised into args.err).
template <int VAR>
__device__ __forceinline__ bool deep_lane_solves(const DeepArgs& a, const double2* tab,
                                                 long long col, int k, double ye, double yp,
                                                 double guess, double e0, double c0,
                                                 double& re, double& rp, int& work) {
  const double tol = a.tol;
  const int maxit = a.maxit;
  const double kBig = 0x1.0p490;
  const bool fastdiv0 =
      a.fast_div_ok && fabs(ye) < kBig && fabs(yp) < kBig && exp_fast_ok(mul(kMC.c005, guess));
  bool fastdiv = fastdiv0;
  double y = ye, t = guess, e = e0, resid = sub(c0, ye);
  int it = 0, pass = 0, order = k;
  work = 0;
  if (!is_finite(ye)) { raise_failure(a.err, col, order, kFailInput); return false; }
  for (;;) {
    if (it > maxit) { raise_failure(a.err, col, order, kFailNoConv); return false; }
    if (fabs(resid) <= tol) {
      work += it;
      if (pass == 1) { rp = t; return true; }
      re = t;
      pass = 1;
      order = a.L + k;
      it = 0;
      y = yp;
      t = guess;
      e = e0;
      fastdiv = fastdiv0;
      if (!is_finite(yp)) { raise_failure(a.err, col, order, kFailInput); return false; }
      resid = sub(c0, yp);
      continue;
    }
    const double deriv = add(mul(kMC.c005, e), kMC.c001);
    t = sub(t, fastdiv ? div_fast(resid, deriv) : div_rn(resid, deriv));
    bool fast;
    if (VAR == kVarApprox) {
      if (!is_finite(t)) { raise_failure(a.err, col, order, kFailDiverged); return false; }
      e = approx_exp_ref(mul(kMC.c005, t));
      fast = false;
    } else {
      const double x = mul(kMC.c005, t);
      fast = exp_fast_ok(x);
      if (fast) {
        e = exp_tang(x, tab);
      } else {
        if (!is_finite(t)) { raise_failure(a.err, col, order, kFailDiverged); return false; }
        e = exp(x);
      }
    }
    resid = sub(add(e, mul(kMC.c001, t)), y);
    fastdiv = fastdiv && fast;
    ++it;
  }
}

template <int VAR>
__global__ void __launch_bounds__(512, 2) deep_kernel(DeepArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* s_tab = reinterpret_cast<double2*>(smem_raw);                 // 512 x 16 B
  double* s_term = reinterpret_cast<double*>(s_tab + kExpTableSize);      // cpb*L
  int* s_work = reinterpret_cast<int*>(s_term + a.cpb * a.L);            // cpb*L
  int* s_col = s_work + a.cpb * a.L;                                      // cpb
  __shared__ int s_tile;

  if (VAR != kVarApprox) {
    for (int i = threadIdx.x; i < kExpTableSize; i += blockDim.x) s_tab[i] = a.exp_tab[i];
  }
  const int L = a.L, cpb = a.cpb;
  const int lanes = cpb * L;
  const int lc = threadIdx.x / L, k = threadIdx.x - (threadIdx.x / L) * L;
  const long long A = *a.count;
  const bool reduced = (VAR == kVarReduced);

  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(a.tile_cursor, 1);
    __syncthreads();
    const long long first = (long long)s_tile * cpb;
    if (first >= A) break;
    if (threadIdx.x < cpb) s_col[threadIdx.x] = (first + threadIdx.x < A) ? a.idx[first + threadIdx.x] : -1;
    __syncthreads();

    double term = 0.0;
    int wl = 0;
    const int c = (threadIdx.x < lanes) ? s_col[lc] : -1;
    if (c >= 0) {
      const double sc = a.s[c];
      const double T = a.T[(long long)k * a.ld_in + c];
      const double q = a.q[(long long)k * a.ld_in + c];
      // physics.cpp:121 / :127 / :146-148 / :155-156
      const double guess = add(24.0, mul(160.0, sc));
      const double rho = add(1.0, mul(kMC.c005, sc));
      const double m = reduced ? div_rn(q, mul(rho, rho)) : div_rn(div_rn(q, rho), rho);
      const double ye = add(add(1.0, mul(1.0e-3, T)), mul(0.1, m));
      const double yp = add(add(add(1.0, mul(8.0e-4, T)), mul(kMC.c005, m)), mul(0.1, sc));
      bool f0;
      const double e0 = deep_exp<VAR>(mul(kMC.c005, guess), s_tab, f0);
      const double c0 = add(e0, mul(kMC.c001, guess));
      double re = 0.0, rp = 0.0;
      const long long col = a.first_col + c;
      if (deep_lane_solves<VAR>(a, s_tab, col, k, ye, yp, guess, e0, c0, re, rp, wl)) {
        // physics.cpp:151-152 / :159-161
        const long long o = (long long)k * a.ld_out + c;
        a.tend_T[o] = add(mul(0.02, sub(add(250.0, mul(2.0, re)), T)),
                          mul(0.3, sin(add(mul(6.0, T), mul(50.0, q)))));
        a.tend_q[o] = mul(kMC.c005, sub(add(kMC.c001, mul(0.002, sin(mul(3.0, rp)))), q));
        term = mul(q, max0(sub(rp, 4.5)));
      }
    }
    if (threadIdx.x < lanes) {
      s_term[threadIdx.x] = term;
      s_work[threadIdx.x] = wl;
    }
    __syncthreads();
    if (threadIdx.x < cpb) {
      const int cc = s_col[threadIdx.x];
      if (cc >= 0) {
        double pr = 0.0;  // ordered k sum, physics.cpp:161
        long long w = 0;
        for (int kk = 0; kk < L; ++kk) {
          pr = add(pr, s_term[threadIdx.x * L + kk]);
          w += s_work[threadIdx.x * L + kk];
        }
        a.precip[cc] = pr;
        a.work[cc] = w;
        a.exited[cc] = 0;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Shallow scheme + deep zero-fill.  The four phase sums of physics.cpp:
// 182-204 depend only on (T, q, s), not on acc, so one streaming pass over
// the levels accumulates all four (each in k order, bit-identical to the
// reference's per-phase loops); the exit predicates (:205-211) then run on
// scalars.  Survivors re-read their rows for the outputs (:214-224).
struct ShallowArgs {
  const double* s;
  const double* T;
  const double* q;
  long long ld_in;
  long long n;
  // shallow outputs
  double* tend_T;
  double* tend_q;
  double* precip;
  long long* work;
  uint8_t* exited;
  long long ld_out;
  // deep outputs (zero-filled for s <= thr)
  double* d_tend_T;
  double* d_tend_q;
  double* d_precip;
  long long* d_work;
  uint8_t* d_exited;
  long long d_ld_out;
  unsigned long long* err;
  const double2* exp_tab;
  long long first_col;
  double thr;
  int L;
};

template <int VAR, bool DO_SHALLOW, bool DO_DEEP_ZERO>
__global__ void __launch_bounds__(256) shallow_kernel(ShallowArgs a) {
  __shared__ double2 s_tab[kExpTableSize];
  if (DO_SHALLOW && VAR != kVarApprox) {
    for (int i = threadIdx.x; i < kExpTableSize; i += blockDim.x) s_tab[i] = a.exp_tab[i];
    __syncthreads();
  }
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.n) return;
  const int L = a.L;
  const double sc = a.s[c];
  if (DO_DEEP_ZERO && !(sc > a.thr)) {
    for (int k = 0; k < L; ++k) {
      a.d_tend_T[(long long)k * a.d_ld_out + c] = 0.0;
      a.d_tend_q[(long long)k * a.d_ld_out + c] = 0.0;
    }
    a.d_precip[c] = 0.0;
    a.d_work[c] = 0;
    a.d_exited[c] = 1;
  }
  if (!DO_SHALLOW) return;
  if (!is_finite(sc)) { raise_failure(a.err, a.first_col + c, 0, kFailActivity); return; }

  // physics.cpp:174-176 weights; 1.0e-3 * w1[j] is formed first (left to
  // right, :186) and rounded exactly as the reference's constant product.
  const double a1_0 = mul(1.0e-3, 0.8), a1_1 = mul(1.0e-3, 1.1), a1_2 = mul(1.0e-3, 0.9),
               a1_3 = mul(1.0e-3, 1.2);
  const bool reduced = (VAR == kVarReduced);
  const double rho = add(1.0, mul(kMC.c005, sc));
  const double rho2 = mul(rho, rho);
  double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
  for (int k = 0; k < L; ++k) {
    const double T = a.T[(long long)k * a.ld_in + c];
    const double q = a.q[(long long)k * a.ld_in + c];
    const double m = reduced ? div_rn(q, rho2) : div_rn(div_rn(q, rho), rho);
    const double x = mul(-50.0, q);
    double ex;
    if (VAR == kVarApprox) ex = approx_exp_ref(x);
    else ex = exp_fast_ok(x) ? exp_tang(x, s_tab) : exp(x);
    p0 = add(p0, add(mul(a1_0, T), mul(30.0, m)));
    p1 = add(p1, add(add(mul(a1_1, T), mul(20.0, m)), mul(0.02, ex)));
    p2 = add(p2, add(mul(a1_2, T), mul(40.0, m)));
    p3 = add(p3, add(mul(a1_3, T), mul(25.0, m)));
  }
  const double dl = (double)L;
  const double ps[4] = {p0, p1, p2, p3};
  const double w3[4] = {0.5, 0.3, 0.4, 0.2};
  const double theta[4] = {0.15, 0.30, 0.45, 0.60};
  double acc = 0.0;
  int phases = 0;
  bool survived = true;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    acc = add(acc, add(div_rn(ps[j], dl), mul(w3[j], sc)));
    ++phases;
    const double lhs = mul(sc, add(1.0, mul(kMC.c005, sin(mul(3.0, acc)))));
    if (lhs < theta[j]) { survived = false; break; }
  }
  a.work[c] = (long long)phases * L;
  if (!survived) {
    for (int k = 0; k < L; ++k) {
      a.tend_T[(long long)k * a.ld_out + c] = 0.0;
      a.tend_q[(long long)k * a.ld_out + c] = 0.0;
    }
    a.precip[c] = 0.0;
    a.exited[c] = 1;
    return;
  }
  const double sa = sin(acc);
  const double base = add(256.0, mul(2.0, sa));
  for (int k = 0; k < L; ++k) {
    const double T = a.T[(long long)k * a.ld_in + c];
    const double q = a.q[(long long)k * a.ld_in + c];
    a.tend_T[(long long)k * a.ld_out + c] = mul(0.005, sub(base, T));
    a.tend_q[(long long)k * a.ld_out + c] = mul(0.02, sub(0.012, q));
  }
  a.precip[c] = mul(sub(sc, 0.5), max0(add(sa, 0.5)));
  a.exited[c] = 0;
}

// ---------------------------------------------------------------------------
// Batched inverse-entropy solve (physics.cpp:101-104), one thread per pair.
template <int VAR>
__global__ void ientropy_kernel(const double* __restrict__ y, const double* __restrict__ g,
                                long long n, double tol, int maxit, double* __restrict__ root,
                                int* __restrict__ iters, unsigned long long* err,
                                const double2* __restrict__ exp_tab) {
  __shared__ double2 s_tab[kExpTableSize];
  if (VAR != kVarApprox) {
    for (int i = threadIdx.x; i < kExpTableSize; i += blockDim.x) s_tab[i] = exp_tab[i];
    __syncthreads();
  }
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double yy = y[i], guess = g[i];
  if (!is_finite(yy) || !is_finite(guess)) { raise_failure(err, i, 0, kFailInput); return; }
  bool f;
  double t = guess;
  double e = deep_exp<VAR>(mul(kMC.c005, t), s_tab, f);
  double resid = sub(add(e, mul(kMC.c001, t)), yy);
  for (int it = 0; it <= maxit; ++it) {
    if (fabs(resid) <= tol) { root[i] = t; iters[i] = it; return; }
    const double deriv = add(mul(kMC.c005, e), kMC.c001);
    t = sub(t, div_rn(resid, deriv));
    if (!is_finite(t)) { raise_failure(err, i, 0, kFailDiverged); return; }
    e = deep_exp<VAR>(mul(kMC.c005, t), s_tab, f);
    resid = sub(add(e, mul(kMC.c001, t)), yy);
  }
  raise_failure(err, i, 0, kFailNoConv);
}

// FP64 roofline probe: 8 independent DFMA chains per thread.
__global__ void __launch_bounds__(256) dfma_probe_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void approx_exp_kernel(const double* __restrict__ x, double* __restrict__ o, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = approx_exp_ref(x[i]);
}

}  // namespace cvg
