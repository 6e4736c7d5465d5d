// convgpu_kernels.cuh -- sm_100a kernels of the convection column path.
//
//   trigger_groups_kernel   deep trigger s > thr (physics.cpp:108-113) with
//                           warp-ballot / block-scan stream compaction into a
//                           dense list of 4-column groups holding a triggered
//                           column (replaces the reference's dynamic
//                           scheduling, sched.cpp:166-173)
//   deep_kernel             deep plume (physics.cpp:106-166) over the group
//                           list: one warp per column, one lane per level,
//                           each lane running its level's entrainment and
//                           precipitation Newton solves (physics.cpp:64-87) in
//                           lockstep; persistent warps claim groups
//                           dynamically, stage the next column with cp.async
//                           and write each group's outputs as whole sectors
//   shallow_kernel          shallow scheme (physics.cpp:168-225), one thread
//                           per column, streaming level-major rows, together
//                           with the zero-fill of groups without a triggered
//                           column (physics.cpp:89-97, :111-113)
//   ientropy_kernel         batched ientropy_solve (physics.cpp:101-104)
//   approx_exp_kernel       approx_exp (physics.cpp:40-60)
//
// Layout: level-major SoA, field[k * ld + c].  The strict path performs every
// IEEE operation of the reference as one uncontracted, correctly rounded
// device operation (colmath.cuh); the relaxed path (default for the variants
// whose reference calls libm exp) differs from it only by rounding noise
// inside the parity window (colmath.cuh, newton_relaxed_step).
#pragma once
#include <cstdint>

#include "bulkcopy.cuh"
#include "colmath.cuh"

namespace cvg {

enum : int { kVarExact = 0, kVarReduced = 1, kVarApprox = 2 };

// Phase-clock instrumentation of the deep worker (debug builds with
// -DCVG_PHASE_CLOCKS only): per-phase SM cycles summed over warps.
// Accumulated per block in shared memory (flushed once per block at the
// kernel's end): per-column global atomics on 8 addresses from every warp
// slowed the instrumented kernel 2.6x and distorted the split.
#ifdef CVG_PHASE_CLOCKS
__device__ unsigned long long g_phase[8];
__shared__ unsigned long long s_phase[8];
#define CVG_PCLK(v) const long long v = clock64()
#define CVG_PACC(i, a, b) if (lane == 0) atomicAdd(&s_phase[i], (unsigned long long)((b) - (a)))
#else
#define CVG_PCLK(v)
#define CVG_PACC(i, a, b)
#endif
enum : int { kFailNone = 0, kFailActivity = 1, kFailInput = 2, kFailDiverged = 3, kFailNoConv = 4 };

// Failure key: lowest column first, then the solve order the serial
// reference would have met (entrainment k, then precipitation k), then kind.
__device__ __forceinline__ void raise_failure(unsigned long long* err, long long col, int order,
                                              int kind) {
  const unsigned long long key =
      ((unsigned long long)col << 16) | ((unsigned long long)order << 3) | (unsigned long long)kind;
  asm volatile("red.relaxed.gpu.global.min.u64 [%0], %1;" ::"l"(err), "l"(key) : "memory");
}

__device__ __forceinline__ double max0(double x) { return (0.0 < x) ? x : 0.0; }

// ---------------------------------------------------------------------------
// Trigger + stream compaction into column GROUPS.  A group is 4 consecutive
// columns -- one 32-byte sector of every level row -- and the list holds
// each group with at least one triggered column as (group << 4) | mask.  The
// deep kernel works through a group's triggered columns and writes the
// group's deep outputs as whole sectors (zeros for its untriggered
// columns); the shallow kernel zero-fills only groups without a triggered
// column.  Per-column 8-byte stores of the deep outputs were partial-sector
// writes (read-modify-write in L2/DRAM) and bounded the deep kernel.
// One thread per group (4 coalesced loads of s), warp ballot + block scan,
// one atomicAdd per block reserves the block's slice; counts[0] = groups,
// counts[1] = triggered columns.
constexpr int kTrigThreads = 256;
constexpr int kGroupCols = 4;

// Per-call words of a workspace reset in one launch (instead of three
// memsets): counts, cursors to 0, failure keys to "none".
__global__ void reset_call_words_kernel(int* counts, int n_counts, unsigned long long* cursor, int n_cursor,
                                        unsigned long long* err, int n_err) {
  const int t = threadIdx.x;
  if (t < n_counts) counts[t] = 0;
  if (t < n_cursor) cursor[t] = 0;
  if (t < n_err) err[t] = ~0ULL;
}

__global__ void __launch_bounds__(kTrigThreads)
trigger_groups_kernel(const double* __restrict__ s, long long n, double thr, long long first_col,
                      long long* __restrict__ groups, int* __restrict__ counts,
                      unsigned long long* __restrict__ err_deep) {
  constexpr int kWarps = kTrigThreads / 32;
  __shared__ int s_wsum[kWarps];
  __shared__ int s_cols[kWarps];
  __shared__ int s_base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long g = (long long)blockIdx.x * kTrigThreads + threadIdx.x;
  unsigned m = 0;
#pragma unroll
  for (int i = 0; i < kGroupCols; ++i) {
    const long long c = g * kGroupCols + i;
    if (c < n) {
      const double sc = s[c];
      if (!is_finite(sc)) raise_failure(err_deep, first_col + c, 0, kFailActivity);
      if (sc > thr) m |= 1u << i;
    }
  }
  const unsigned bal = __ballot_sync(0xffffffffu, m != 0);
  const int ncols = __reduce_add_sync(0xffffffffu, __popc(m));
  if (lane == 0) {
    s_wsum[warp] = __popc(bal);
    s_cols[warp] = ncols;
  }
  __syncthreads();
  if (warp == 0) {
    const int v = lane < kWarps ? s_wsum[lane] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < kWarps; o <<= 1) {
      const int x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    const int cols = __reduce_add_sync(0xffffffffu, lane < kWarps ? s_cols[lane] : 0);
    if (lane < kWarps) s_wsum[lane] = incl - v;
    if (lane == kWarps - 1) {
      s_base = incl > 0 ? atomicAdd(&counts[0], incl) : 0;
      if (cols > 0) atomicAdd(&counts[1], cols);
    }
  }
  __syncthreads();
  if (m) groups[s_base + s_wsum[warp] + __popc(bal & ((1u << lane) - 1u))] = (g << 4) | (long long)m;
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
  const long long* groups;  // compacted groups with a triggered column: (group << 4) | mask
  unsigned long long* trace;  // optional [grid][3]: smid, start, end (globaltimer ns)
  const int* count;       // number of listed groups (device)
  long long n;            // columns
  unsigned long long* cursor;  // [0] work cursor (zeroed per call), [1..32] dummies
  unsigned long long* err;
  const double2* exp_tab; // 2^(j/512) double-double table (global)
  long long first_col;
  double thr, tol;
  int maxit;
  int L;                  // levels
  bool fast_div_ok;       // newton_tol >= 2^-500
  bool relaxed;           // relaxed-rounding Newton update allowed (colmath.cuh)
  bool far32;             // FP32 far phase allowed (relaxed only; colmath.cuh)
  int y_win;              // far_window_limit(): hi-word bound of the hot path's targets
  bool tree_precip;       // precip summed as a warp tree (relaxed path; else k order)
  bool vec4;              // outputs 32-byte aligned with ld_out % 4 == 0 (group stores)
};

// Deep-kernel lanes read a lane-private copy of the exp table (see
// exp_tang); other kernels pass the plain table with kTabCopies = 1 views.
constexpr int kTabCopies = 1;

template <int VAR, int STRIDE = kTabCopies>
__device__ __forceinline__ double deep_exp(double x, const double2* tab) {
  if (VAR == kVarApprox) return approx_exp_ref(x);
  return exp_fast_ok(x) ? exp_tang<STRIDE>(x, tab) : exp_cold(x);
}

// Fast-path exp for |x| < 340 (caller checked exp_fast_ok): the table exp,
// or approx_exp with its ldexp as an exact exponent add (|k| <= 491).
template <int VAR>
__device__ __forceinline__ double deep_exp005_fast(double t, const double2* tab) {
  if (VAR == kVarApprox) return approx_exp_ref_fast(mul(kMC.c005, t));
  return exp005_tang<kTabCopies>(t, tab);
}

// Reference-faithful Newton loop (physics.cpp:64-87) continued from any
// state, with every range check: convergence tested before each update, at
// most max_iter updates, non-finite iterates rejected, IEEE division and
// full-range exp.  `it` counts updates already taken.  Returns false on
// failure (raised into a.err with the solve's reference order).
template <int VAR>
__device__ __forceinline__ bool newton_generic(const DeepArgs& a, const double2* tab, long long col,
                                            int order, double y, double& t, double& e,
                                            double& resid, int& it) {
  for (;;) {
    if (it > a.maxit) { raise_failure(a.err, col, order, kFailNoConv); return false; }
    if (fabs(resid) <= a.tol) return true;
    const double deriv = add(mul(kMC.c005, e), kMC.c001);
    t = sub(t, div_rn(resid, deriv));
    if (!is_finite(t)) { raise_failure(a.err, col, order, kFailDiverged); return false; }
    e = deep_exp<VAR>(mul(kMC.c005, t), tab);
    resid = sub(add(e, mul(kMC.c001, t)), y);
    ++it;
  }
}

// Completes one solve: the common case (converged, within max_iter) inline,
// anything else in the cold generic loop.
template <int VAR>
__device__ __forceinline__ bool newton_finish(const DeepArgs& a, const double2* tab, long long col,
                                              int order, double y, double& t, double& e, double& h,
                                              int& it) {
  if (it <= a.maxit && fabs(h) <= a.tol) return true;
  return newton_generic<VAR>(a, tab, col, order, y, t, e, h, it);
}

// The lane's two solves -- entrainment (reference order k) and
// precipitation (order L + k) of level k -- iterate in lockstep: two
// independent dependency chains per lane (ILP 2) in one straight-line loop.
// Within a column the two solves' iteration counts agree on ~99% of levels
// (the guess is shared), so the loop runs while BOTH are unconverged and
// hands whichever is left (usually nothing, at most an update or two) to
// newton_finish.
//
// The fast loop carries no per-update range checks.  Its precondition P:
//   newton_tol >= 2^-500, -60 < y < 2^490 for both solves, |0.05 guess| <
//   340, and the guess right of both roots (initial residuals > 0).
// f(t) = exp(0.05 t) + 0.01 t is increasing and convex, so Newton from the
// right descends monotonically onto the root and never overshoots it (an FP
// step's relative error ~1e-15 can only cross the root within ~1e-13 of
// it); every iterate therefore lies in [root - tiny, guess].  y > -60 gives
// root > 100 (y - 1) > -6100, so |0.05 t| < 340 throughout: exp_tang's
// domain.  Then every derivative 0.05 e + 0.01 lies in [0.01, 2^488) and
// every residual divided (only while |r| > tol) in (2^-500, 2^500): the
// operand range where div_fast is exact.  Inputs outside P take the
// reference-faithful generic loop from the start.  Semantics per solve are
// exactly the reference's; a failure in one solve does not stop the other
// (the reference reports the first failure in its own solve order,
// recovered from the failure key).
template <int VAR>
__device__ __forceinline__ bool deep_lane_pair(const DeepArgs& a, const double2* tab, unsigned tab1_addr,
                                               long long col,
                                               int k, double ye, double yp, double guess, double e0,
                                               double c0, bool col_far, double& re, double& rp, int& work) {
  const double kBig = 0x1.0p490;
  double te = guess, ee = e0, he = sub(c0, ye);
  double tp = guess, ep = e0, hp = sub(c0, yp);
  int it = 0;
  const int maxit = a.maxit;
  if (VAR != kVarApprox && col_far && in_far_window(ye, a.y_win) && in_far_window(yp, a.y_win) &&
      min(hi_word(he), hi_word(hp)) > 0) {
    // Hot path.  The window (host-computed, far_window_limit) guarantees
    // the fast-loop precondition P and relaxed_ok for both targets; the
    // guess is right of both roots (residuals > 0).  FP32 far phase
    // (colmath.cuh) while both |h| > kFar32H, then exp and h re-evaluated
    // in FP64 at the FP32 iterates and the relaxed FP64 update to the end.
    const double tol = a.tol;
    int left = maxit + 1;   // updates still allowed (the loop may take one
                            // more than maxit; newton_finish then fails it)
    CVG_PCLK(pf0);
    {
      float fte = (float)guess, ftp = fte, fee = (float)e0, fep = fee;
      float fhe = (float)he, fhp = (float)hp;
      const float fye = (float)ye, fyp = (float)yp;
      while (left > 0 && fminf(fabsf(fhe), fabsf(fhp)) > kFar32H) {
        newton_far32_step(fte, fee, fhe, fye);
        newton_far32_step(ftp, fep, fhp, fyp);
        --left;
      }
      te = fte;
      tp = ftp;
    }
#ifdef CVG_PHASE_CLOCKS
    {
      CVG_PCLK(pf1);
      const int lane = threadIdx.x & 31;
      CVG_PACC(5, pf0, pf1);   // FP32 far loop
    }
#endif
    ee = exp_relaxed1(kRC, te, tab1_addr);
    ep = exp_relaxed1(kRC, tp, tab1_addr);
    he = fma(kMC.c001, te, ee - ye);
    hp = fma(kMC.c001, tp, ep - yp);
    if (min(hi_word(he), hi_word(hp)) <= 0) {
      // left of a root (not expected: the switch happens O(1) away from
      // it): redo both solves from the guess with the FP64 update
      te = tp = guess;
      ee = ep = e0;
      he = sub(c0, ye);
      hp = sub(c0, yp);
      left = maxit + 1;
    }
    CVG_PCLK(pl0);
    if (left > 0) do {
      if (abs_le_either(he, hp, tol)) break;
      newton_relaxed_step(te, ee, he, ye, tab1_addr);
      newton_relaxed_step(tp, ep, hp, yp, tab1_addr);
    } while (--left != 0);
    it = maxit + 1 - max(left, 0);
#ifdef CVG_PHASE_CLOCKS
    {
      CVG_PCLK(pl1);
      const int lane = threadIdx.x & 31;
      CVG_PACC(4, pl0, pl1);   // relaxed Newton loop
    }
#endif
    int ie = it, ip = it;
    bool ok = newton_finish<VAR>(a, tab, col, k, ye, te, ee, he, ie);
    if (!newton_finish<VAR>(a, tab, col, a.L + k, yp, tp, ep, hp, ip)) ok = false;
    re = te;
    rp = tp;
    work = ie + ip;
    return ok;
  }
  const bool inputs_ok = is_finite(ye) && is_finite(yp);
  const bool fast_ok = inputs_ok && a.fast_div_ok && ye > -60.0 && yp > -60.0 && ye < kBig &&
                       yp < kBig && he > 0.0 && hp > 0.0 && exp_fast_ok(mul(kMC.c005, guess));
  if (VAR != kVarApprox && fast_ok && a.relaxed && relaxed_ok(ye, a.tol) && relaxed_ok(yp, a.tol)) {
    // relaxed update (colmath.cuh): same iteration and stop test, rounding
    // noise only; the exact sequence below is the one the reference runs
    const double tol = a.tol;
    int left = maxit + 1;
    if (left > 0) do {
      if (abs_le_either(he, hp, tol)) break;
      newton_relaxed_step(te, ee, he, ye, tab1_addr);
      newton_relaxed_step(tp, ep, hp, yp, tab1_addr);
    } while (--left != 0);
    it = maxit + 1 - max(left, 0);
  } else if (fast_ok) {
    const double tol = a.tol;
    while (it <= maxit) {
      if (abs_le(he, tol) || abs_le(hp, tol)) break;   // tol >= 2^-500 here
      te = sub(te, div_fast(he, add(mul(kMC.c005, ee), kMC.c001)));
      tp = sub(tp, div_fast(hp, add(mul(kMC.c005, ep), kMC.c001)));
      ee = deep_exp005_fast<VAR>(te, tab);
      ep = deep_exp005_fast<VAR>(tp, tab);
      he = sub(add(ee, mul(kMC.c001, te)), ye);
      hp = sub(add(ep, mul(kMC.c001, tp)), yp);
      ++it;
    }
  }
  int ie = it, ip = it;
  bool ok = true;
  if (!inputs_ok) {
    if (!is_finite(ye)) { raise_failure(a.err, col, k, kFailInput); ok = false; }
    else if (!newton_generic<VAR>(a, tab, col, k, ye, te, ee, he, ie)) ok = false;
    if (!is_finite(yp)) { raise_failure(a.err, col, a.L + k, kFailInput); ok = false; }
    else if (!newton_generic<VAR>(a, tab, col, a.L + k, yp, tp, ep, hp, ip)) ok = false;
  } else {
    if (!newton_finish<VAR>(a, tab, col, k, ye, te, ee, he, ie)) ok = false;
    if (!newton_finish<VAR>(a, tab, col, a.L + k, yp, tp, ep, hp, ip)) ok = false;
  }
  re = te;
  rp = tp;
  work = ie + ip;
  return ok;
}

// One level (lane) of a triggered column: physics.cpp:140-161 for level k --
// m = q / rho / rho (physics.hpp:94-96, shared-divisor form of div_rn), the
// entrainment and precipitation solves (deep_lane_pair), the tendencies and
// the precipitation term.  Returns false on a numeric failure (outputs 0).
template <int VAR>
__device__ __forceinline__ bool deep_level(const DeepArgs& a, const double2* s_tab, unsigned tab1_addr,
                                           long long col, int k, double sc, double rho, double guess,
                                           double e0, double c0, bool col_far, double T, double q,
                                           double& tT, double& tq, double& term, int& w) {
  const bool reduced = (VAR == kVarReduced);
  double m_;
  {
    const double dv = reduced ? mul(rho, rho) : rho;
    if (div_operand_ok(dv) && div_operand_ok(q)) {
      const double ydv = rcp_refined(dv);
      m_ = div_by(q, dv, ydv);
      if (!reduced) m_ = div_operand_ok(m_) ? div_by(m_, dv, ydv) : div_rn(m_, dv);
    } else {
      m_ = reduced ? div_rn(q, dv) : div_rn(div_rn(q, rho), rho);
    }
  }
  // physics.cpp:147-148 / :156-157
  const double ye = add(add(1.0, mul(1.0e-3, T)), mul(0.1, m_));
  const double yp = add(add(add(1.0, mul(8.0e-4, T)), mul(kMC.c005, m_)), mul(0.1, sc));
  double re = 0.0, rp = 0.0;
  w = 0;
  term = tT = tq = 0.0;
  if (!deep_lane_pair<VAR>(a, s_tab, tab1_addr, col, k, ye, yp, guess, e0, c0, col_far, re, rp, w)) return false;
  // physics.cpp:151-152 / :159-161
  double sin_a, sin_b;
  sin2_cw(add(mul(6.0, T), mul(50.0, q)), mul(3.0, rp), sin_a, sin_b);
  tT = add(mul(0.02, sub(add(250.0, mul(2.0, re)), T)), mul(0.3, sin_a));
  tq = mul(kMC.c005, sub(add(kMC.c001, mul(0.002, sin_b)), q));
  term = mul(q, max0(sub(rp, 4.5)));
  return true;
}

// One warp per triggered column, lane k = level k (levels k, k+32, ... when
// L > 32).  A column's 60 solves share the guess, so their iteration counts
// agree almost everywhere and the warp runs converged (0.03 mean spread);
// the trigger kernel's s-bucketing keeps a warp's consecutive entries at
// near-equal work, and warps never wait on a block barrier.  Per-column scalars are finished in batches: each column's
// precipitation terms are parked in shared memory and, every kBatch
// columns, lane i sums column i's terms in k order (physics.cpp:161) -- one
// warp instruction serves kBatch columns instead of one.
constexpr int kDeepChunk = 1;   // list entries (groups) claimed per atomic (power of 2)

// Issued by lane 0 only, at cursor + lane (= cursor): an address ptxas
// cannot prove warp-uniform, so it does not rewrite the atomic into its
// aggregated form (vote + one atomic + SHFL of the result), whose SHFL
// would wait for the atomic on the spot.
__device__ __forceinline__ long long claim_chunk(unsigned long long* cursor_plus_lane) {
  unsigned long long r;
  asm volatile("atom.global.add.u64 %0, [%1], %2;" : "=l"(r) : "l"(cursor_plus_lane), "n"(kDeepChunk) : "memory");
  return (long long)r;
}

// The group's per-column scalars live in s_gwork / s_gok / s_gpr [4].
// Per-warp shared scratch of the deep worker, in doubles:
//   NARROW: [32] (two group-entry slots, padded), group outputs tend_T,
//           tend_q [4][32] each, precip terms [4][32]
//   wide:   precip terms [L] of the current column
__host__ __device__ constexpr int deep_warp_doubles(bool narrow, int L) {
  return narrow ? 32 + 3 * kGroupCols * 32 : L;
}

// The deep role of a warp: walks the group list until it is exhausted.
// s_tab points at this lane's copy of the replicated exp table; s_warp is
// this warp's scratch (deep_warp_doubles), s_gwork / s_gok the group's
// per-column work counts and success flags.
template <int VAR, bool NARROW>
__device__ __forceinline__ void deep_worker(const DeepArgs& a, const double2* s_tab, unsigned tab1_addr,
                                            double* s_warp, int* s_gwork, int* s_gok, double* s_gpr, int lane) {
  const int L = a.L;
  const long long G = *a.count;
  // Work distribution: warps claim groups from a global cursor (one atomic
  // per group, a group ahead), so SMs finish together whatever the
  // per-column cost mix.  Software pipeline: a column's (s, T[lane],
  // q[lane]) are staged during the previous column's solves, the next
  // group's entry is known a group ahead, the one after it is loaded then.
  // Lane 0 alone issues the claim, as inline PTX: the compiler's
  // warp-aggregated atomicAdd would broadcast the result (SHFL) right away
  // and so wait for the atomic; here the result stays in lane 0 until the
  // group after next needs it.
  long long next_raw = 0;
  const unsigned lane_op = opaque_u32(lane);
  auto claim = [&]() { if (lane == 0) next_raw = claim_chunk(a.cursor + lane_op); };
  auto advance = [&](long long x) -> long long {
    if (((x + 1) & (kDeepChunk - 1)) != 0) return x + 1;
    const long long r = __shfl_sync(0xffffffffu, next_raw, 0);
    claim();
    return r;
  };
  auto entry = [&](long long x) -> long long { return x < G ? a.groups[x] : -1; };
  claim();
  long long j = __shfl_sync(0xffffffffu, next_raw, 0);
  claim();
  long long jn = advance(j);
  long long e = entry(j), en = entry(jn);
  long long jnn = jn < G ? advance(jn) : G;
  // NARROW: the entry after next arrives by cp.async into one of two
  // per-warp shared slots (the first doubles of the warp's scratch), so no register
  // waits for it -- a plain load's result had to be copied into the
  // rotating entry registers right away, and that copy stalled on the load
  // (5 % of the kernel's warp samples)
  const unsigned ent_addr = smem_u32(s_warp);
  int eslot = 0;
  auto fetch_entry = [&](long long x) {
    if (lane == 0) {
      const unsigned d = ent_addr + 8 * eslot;
      if (x < G) cp_async8_u32(d, a.groups + x);
      else asm volatile("st.shared.s64 [%0], %1;" ::"r"(d), "l"(-1LL) : "memory");
      cp_async_commit();
    }
  };
  auto take_entry = [&]() -> long long {
    if (lane == 0) cp_async_wait_all();
    __syncwarp();
    long long v;
    asm volatile("ld.shared.s64 %0, [%1];" : "=l"(v) : "r"(ent_addr + 8 * eslot) : "memory");
    eslot ^= 1;
    return v;
  };
  long long enn = 0;
  if (NARROW) fetch_entry(jnn);
  else enn = entry(jnn);
  double* s_outT = s_warp + 32;   // NARROW: [4][32] (s_warp[0..1]: group entry slots)
  double* s_outQ = s_outT + kGroupCols * 32;
  double* s_term = NARROW ? s_outQ + kGroupCols * 32 : s_warp;   // NARROW: [4][32]; wide: [L]
  // this lane's level rows (lane < L)
  const double* T_row = a.T + (long long)min(lane, L - 1) * a.ld_in;
  const double* q_row = a.q + (long long)min(lane, L - 1) * a.ld_in;
  double* outT_row = a.tend_T + (long long)min(lane, L - 1) * a.ld_out;
  double* outQ_row = a.tend_q + (long long)min(lane, L - 1) * a.ld_out;
  // NARROW: the next column's (s, T[lane], q[lane]) are prefetched into
  // registers with read-only loads during the current column (cp.async
  // staging into shared memory measured the same and cost LDGSTS bank
  // conflicts)
  double nx_s = 0.0, nx_T = 0.0, nx_q = 0.0;
  auto prefetch = [&](long long cc) {
    nx_s = __ldg(a.s + cc);
    if (lane < L) {
      nx_T = __ldg(T_row + cc);
      nx_q = __ldg(q_row + cc);
    }
  };
  if (e >= 0) {
  long long g = e >> 4;
  unsigned m = (unsigned)(e & 15), rem = m;
  int i = __ffs(rem) - 1;
  rem &= rem - 1;
  long long c = g * kGroupCols + i;
  if (NARROW) prefetch(c);
  for (;;) {
    CVG_PCLK(ph0);
    // the column after this one: the group's next, or the next group's first
    long long cn = -1;
    if (rem) cn = g * kGroupCols + (__ffs(rem) - 1);
    else if (en >= 0) cn = (en >> 4) * kGroupCols + (__ffs((unsigned)(en & 15)) - 1);
    double sc, T_c = 0.0, q_c = 0.0;
    if (NARROW) {
      sc = nx_s;
      T_c = nx_T;
      q_c = nx_q;
#ifdef CVG_PHASE_CLOCKS
      {
        double chk = sc + T_c + q_c;   // force the staged values here
        asm volatile("" : "+d"(chk));
        CVG_PCLK(phw);
        CVG_PACC(6, ph0, phw);   // wait for the staged column
      }
#endif
      if (cn >= 0) prefetch(cn);
    } else {
      sc = a.s[c];
    }
    // physics.cpp:121 / :127 / :146
    const double guess = add(24.0, mul(160.0, sc));
    const double rho = add(1.0, mul(kMC.c005, sc));
    const double e0 = deep_exp<VAR>(mul(kMC.c005, guess), s_tab);
    const double c0 = add(e0, mul(kMC.c001, guess));
    // far phase: guesses below 512 (FP32 ulp of t <= 6e-5, <= ~25 far steps)
    const bool col_far = guess < 512.0;
    CVG_PCLK(ph1);
    const long long col = a.first_col + c;
    int wl = 0;
    bool ok_all = true;
    double term_l = 0.0;
    // NARROW (L <= 32): one level per lane, its (T, q) staged; wide columns
    // loop over levels lane, lane + 32, ... with plain loads
    for (int k = lane; k < L; k += 32) {
      double T, q;
      if (NARROW) {
        T = T_c;
        q = q_c;
      } else {
        T = a.T[(long long)k * a.ld_in + c];
        q = a.q[(long long)k * a.ld_in + c];
      }
      double term, tT, tq;
      int w;
      if (!deep_level<VAR>(a, s_tab, tab1_addr, col, k, sc, rho, guess, e0, c0, col_far, T, q, tT, tq, term, w))
        ok_all = false;
      if (NARROW) {
        s_outT[i * 32 + k] = tT;
        s_outQ[i * 32 + k] = tq;
        if (!a.tree_precip) s_term[i * 32 + k] = term;
        else term_l = term;
      } else {
        a.tend_T[(long long)k * a.ld_out + c] = tT;
        a.tend_q[(long long)k * a.ld_out + c] = tq;
        s_term[k] = term;
      }
      wl += w;
    }
    CVG_PCLK(ph3);
    const int wsum = __reduce_add_sync(0xffffffffu, wl);
    const bool ok = __all_sync(0xffffffffu, ok_all);
    if (NARROW && a.tree_precip) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) term_l = add(term_l, __shfl_xor_sync(0xffffffffu, term_l, o));
      if (lane == 0) s_gpr[i] = term_l;
    }
    if (lane == 0) {
      s_gwork[i] = wsum;
      s_gok[i] = ok;
    }
    __syncwarp();
    if (!NARROW && lane == 0) {   // ordered k sum, physics.cpp:161
      double pr = 0.0;
      for (int kk = 0; kk < L; ++kk) pr = add(pr, s_term[kk]);
      s_gpr[i] = pr;
    }
    if (!NARROW) __syncwarp();   // s_term is reused by the next column
    CVG_PCLK(ph4);
    if (rem == 0) {
      // last triggered column of group g: write the group's deep outputs,
      // zeros for its untriggered columns (physics.cpp:89-97)
      const long long c0g = g * kGroupCols;
      if (NARROW) {
        // lane k writes row k of the group: 4 columns = one 32-byte sector
        if (lane < L) {
          double vT[kGroupCols], vQ[kGroupCols];
#pragma unroll
          for (int ii = 0; ii < kGroupCols; ++ii) {
            const bool trig = (m >> ii) & 1u;
            vT[ii] = trig ? s_outT[ii * 32 + lane] : 0.0;
            vQ[ii] = trig ? s_outQ[ii * 32 + lane] : 0.0;
          }
          double* pT = outT_row + c0g;
          double* pQ = outQ_row + c0g;
          if (a.vec4 && c0g + kGroupCols <= a.n) {
            st_global_v4f64(pT, vT[0], vT[1], vT[2], vT[3]);
            st_global_v4f64(pQ, vQ[0], vQ[1], vQ[2], vQ[3]);
          } else {
#pragma unroll
            for (int ii = 0; ii < kGroupCols; ++ii)
              if (c0g + ii < a.n) {
                pT[ii] = vT[ii];
                pQ[ii] = vQ[ii];
              }
          }
        }
      } else {
        for (int r = lane; r < kGroupCols * L; r += 32) {
          const int k = r / kGroupCols, ii = r % kGroupCols;
          const long long cc = c0g + ii;
          if (cc < a.n && !((m >> ii) & 1u)) {
            a.tend_T[(long long)k * a.ld_out + cc] = 0.0;
            a.tend_q[(long long)k * a.ld_out + cc] = 0.0;
          }
        }
      }
      if (lane < kGroupCols && c0g + lane < a.n) {
        const long long cc = c0g + lane;
        if ((m >> lane) & 1u) {
          double pr = 0.0;
          if (NARROW && !a.tree_precip) {   // ordered k sum, physics.cpp:161
            const double* tt = s_term + lane * 32;
            for (int kk = 0; kk < L; ++kk) pr = add(pr, tt[kk]);
          } else {
            pr = s_gpr[lane];
          }
          if (s_gok[lane]) {
            a.precip[cc] = pr;
            a.work[cc] = s_gwork[lane];
            a.exited[cc] = 0;
          }
        } else {
          a.precip[cc] = 0.0;
          a.work[cc] = 0;
          a.exited[cc] = 1;
        }
      }
      __syncwarp();
      if (en < 0) break;
      // next group; load the entry after it
      e = en;
      en = NARROW ? take_entry() : enn;
      j = jn;
      jn = jnn;
      jnn = jn < G ? advance(jn) : G;
      if (NARROW) fetch_entry(jnn);
      else enn = entry(jnn);
      g = e >> 4;
      m = (unsigned)(e & 15);
      rem = m;
    }
    {
      CVG_PCLK(ph5);
      CVG_PACC(0, ph0, ph1);   // wait + stage + prologue to col
      CVG_PACC(1, ph1, ph3);   // per-level: m, ye/yp, Newton, sin, tendencies
      CVG_PACC(2, ph3, ph4);   // reductions
      CVG_PACC(3, ph4, ph5);   // group flush + advance
    }
    i = __ffs(rem) - 1;
    rem &= rem - 1;
    c = g * kGroupCols + i;
  }
  }   // e >= 0
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
  unsigned long long* trace;  // optional [grid][3]: smid, start, end (globaltimer ns)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// One column of the shallow scheme (and/or the deep zero-fill), one thread.
// STRIDE: exp table layout (1 = plain, kTabCopies = replicated, lane copy).
// The level loop runs in chunks of kShChunk with the chunk's loads issued
// before any use, so each thread keeps 2 kShChunk loads in flight.
constexpr int kShChunk = 5;

// Where a column's (T[k], q[k]) come from: global rows (stride ld) or a
// shared-memory tile (stride = tile width).
struct GlobalRows {
  const double* T;
  const double* q;
  long long ld;
  __device__ __forceinline__ double t(int k) const { return T[(long long)k * ld]; }
  __device__ __forceinline__ double m(int k) const { return q[(long long)k * ld]; }
};

// The deep zero-fill of a column belongs to the shallow kernel only when its
// whole column group has no triggered column (the deep kernel writes every
// column of a triggered group, trigger_groups_kernel).  Callers run with
// lane == column % 32 inside the warp (group = 4 aligned lanes); lanes of
// columns >= n are inactive and count as untriggered.
__device__ __forceinline__ bool group_untriggered(double sc, double thr) {
  const unsigned b = __ballot_sync(__activemask(), sc > thr);
  return ((b >> ((threadIdx.x & 31) & ~(kGroupCols - 1))) & ((1u << kGroupCols) - 1)) == 0;
}

template <int VAR, bool DO_SHALLOW, bool DO_DEEP_ZERO, int STRIDE, class SRC, bool RELAX = false>
__device__ __forceinline__ void shallow_column_src(const ShallowArgs& a, long long c, double sc,
                                                   const SRC& src, const double2* tab, bool zero_deep) {
  const int L = a.L;
  if (DO_DEEP_ZERO && zero_deep) {
#pragma unroll 10
    for (int k = 0; k < L; ++k) {
      __stcs(&a.d_tend_T[(long long)k * a.d_ld_out + c], 0.0);
      __stcs(&a.d_tend_q[(long long)k * a.d_ld_out + c], 0.0);
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
  // the per-level divisions share one divisor: its reciprocal is refined
  // once per column (div_by == div_fast bit for bit)
  const double dv = reduced ? rho2 : rho;
  const bool dv_ok = div_operand_ok(dv);
  const double ydv = rcp_refined(dv);
  double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
  if (RELAX) {
    // Relaxed phase sums (Exact / StrengthReduced; CVG_STRICT=1 keeps the
    // reference's per-term order below).  Each phase sum is linear in the
    // level values: sum_k (a1_j T_k + w2_j q_k / rho^2 [+ 0.02 e^-50q_k])
    // = a1_j sum T + (w2_j / rho^2) sum q [+ 0.02 sum e^-50q], so one pass
    // accumulates three sums and the phases follow from them -- rounding
    // differs from the reference's by ~1e-15 relative, far inside the 1e-10
    // output tolerance and the 1e-9 exit-predicate margin.
    const unsigned tab_addr = (unsigned)__cvta_generic_to_shared(tab);
    double sT = 0.0, sQ = 0.0, sE = 0.0;
    for (int k0 = 0; k0 < L; k0 += kShChunk) {
      double Tk[kShChunk], qk[kShChunk];
#pragma unroll
      for (int i = 0; i < kShChunk; ++i) {
        const int k = k0 + i;
        if (k < L) {
          Tk[i] = src.t(k);
          qk[i] = src.m(k);
        }
      }
#pragma unroll
      for (int i = 0; i < kShChunk; ++i) {
        if (k0 + i >= L) break;
        const double q = qk[i];
        // exp(-50 q): table exp in q units for |q| < 6.5, else libdevice
        const double ex = (__double2hiint(q) & 0x7fffffff) < 0x401a0000 ? exp_relaxed<STRIDE>(kRCq, q, tab_addr)
                                                                         : exp_cold(mul(-50.0, q));
        sT = sT + Tk[i];
        sQ = sQ + q;
        sE = sE + ex;
      }
    }
    const double ir = div_rn(1.0, rho);
    const double sm = sQ * (reduced ? div_rn(1.0, rho2) : ir * ir);
    p0 = fma(a1_0, sT, 30.0 * sm);
    p1 = fma(a1_1, sT, fma(20.0, sm, 0.02 * sE));
    p2 = fma(a1_2, sT, 40.0 * sm);
    p3 = fma(a1_3, sT, 25.0 * sm);
  } else
  for (int k0 = 0; k0 < L; k0 += kShChunk) {
    double Tk[kShChunk], qk[kShChunk];
#pragma unroll
    for (int i = 0; i < kShChunk; ++i) {
      const int k = k0 + i;
      if (k < L) {
        Tk[i] = src.t(k);
        qk[i] = src.m(k);
      }
    }
#pragma unroll
    for (int i = 0; i < kShChunk; ++i) {
      if (k0 + i >= L) break;
      const double T = Tk[i], q = qk[i];
      double m;
      if (dv_ok && div_operand_ok(q)) {
        m = div_by(q, dv, ydv);
        if (!reduced) m = div_operand_ok(m) ? div_by(m, dv, ydv) : div_rn(m, dv);
      } else {
        m = reduced ? div_rn(q, rho2) : div_rn(div_rn(q, rho), rho);
      }
      const double x = mul(-50.0, q);
      double ex;
      if (VAR == kVarApprox) ex = approx_exp_ref(x);
      else ex = exp_fast_ok(x) ? exp_tang<STRIDE>(x, tab) : exp_cold(x);
      p0 = add(p0, add(mul(a1_0, T), mul(30.0, m)));
      p1 = add(p1, add(add(mul(a1_1, T), mul(20.0, m)), mul(0.02, ex)));
      p2 = add(p2, add(mul(a1_2, T), mul(40.0, m)));
      p3 = add(p3, add(mul(a1_3, T), mul(25.0, m)));
    }
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
    const double lhs = mul(sc, add(1.0, mul(kMC.c005, sin_cw(mul(3.0, acc)))));
    if (lhs < theta[j]) { survived = false; break; }
  }
  a.work[c] = (long long)phases * L;
  if (!survived) {
#pragma unroll 10
    for (int k = 0; k < L; ++k) {
      __stcs(&a.tend_T[(long long)k * a.ld_out + c], 0.0);
      __stcs(&a.tend_q[(long long)k * a.ld_out + c], 0.0);
    }
    a.precip[c] = 0.0;
    a.exited[c] = 1;
    return;
  }
  const double sa = sin_cw(acc);
  const double base = add(256.0, mul(2.0, sa));
#pragma unroll 10
  for (int k = 0; k < L; ++k) {
    const double T = src.t(k);
    const double q = src.m(k);
    __stcs(&a.tend_T[(long long)k * a.ld_out + c], mul(0.005, sub(base, T)));
    __stcs(&a.tend_q[(long long)k * a.ld_out + c], mul(0.02, sub(0.012, q)));
  }
  a.precip[c] = mul(sub(sc, 0.5), max0(add(sa, 0.5)));
  a.exited[c] = 0;
}

template <int VAR, bool DO_SHALLOW, bool DO_DEEP_ZERO, int STRIDE, bool RELAX = false>
__device__ __forceinline__ void shallow_column(const ShallowArgs& a, long long c, const double2* tab) {
  const double sc = a.s[c];
  shallow_column_src<VAR, DO_SHALLOW, DO_DEEP_ZERO, STRIDE, GlobalRows, RELAX>(
      a, c, sc, GlobalRows{a.T + c, a.q + c, a.ld_in}, tab, group_untriggered(sc, a.thr));
}

constexpr int kShallowThreads = 128;

// Standalone shallow(+zero-fill) kernel: one thread per column.
template <int VAR, bool DO_SHALLOW, bool DO_DEEP_ZERO, bool RELAX = false, int MINB = 8>
__global__ void __launch_bounds__(kShallowThreads, MINB) shallow_kernel(ShallowArgs a) {
  __shared__ double2 s_tab[kExpTableSize];
  if (DO_SHALLOW && VAR != kVarApprox) {
    for (int i = threadIdx.x; i < kExpTableSize; i += blockDim.x) s_tab[i] = a.exp_tab[i];
    __syncthreads();
  }
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (a.trace && threadIdx.x == 0) {
    a.trace[3 * blockIdx.x] = smid();
    a.trace[3 * blockIdx.x + 1] = gtimer();
  }
  if (c < a.n) shallow_column<VAR, DO_SHALLOW, DO_DEEP_ZERO, 1, RELAX>(a, c, s_tab);
  if (a.trace) {
    __syncthreads();
    if (threadIdx.x == 0) a.trace[3 * blockIdx.x + 2] = gtimer();
  }
}

// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Persistent deep kernel: one block per SM; every warp works the deep list
// (deep_worker).  kDeepWarps when it runs alone, kDeepWarpsOverlap when the
// shallow kernel shares the SMs (convgpu.cu, overlap mode).
// Measured (f02, 1 B200, grouped sector-wide stores): alone, 20 warps (0.478
// ms) beat 16 (0.487) and 24 (0.503, register-capped); in overlap mode 12
// warps leave room for three 128-thread shallow blocks per SM, enough for
// the shallow kernel to finish under the deep one (step 0.66 ms, against
// 0.74 at 14 warps and 0.81 at 16, where the shallow blocks starve).
constexpr int kDeepWarps = 20;
constexpr int kDeepWarpsOverlap = 12;

// Register cap per thread.  Blocks of up to 16 warps run beside the
// shallow kernel (overlap mode): they get the register file minus three
// shallow blocks (3 x 128 threads x 64 registers), so three shallow blocks
// always fit (at 12 warps the uncapped kernel took 107 -> 112 registers and
// left room for two); larger blocks run alone and get the whole file.
template <int NW>
constexpr int deep_max_regs() {
  constexpr int budget = NW <= 16 ? 65536 - 3 * 128 * 64 : 65536;
  return ((budget / (NW * 32)) & ~7) > 255 ? 255 : ((budget / (NW * 32)) & ~7);
}

template <int VAR, bool NARROW, int NW>
__global__ void __maxnreg__(deep_max_regs<NW>()) deep_kernel(DeepArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
#ifdef CVG_PHASE_CLOCKS
  if (threadIdx.x < 8) s_phase[threadIdx.x] = 0;
#endif
  if (a.trace && threadIdx.x == 0) {
    a.trace[3 * blockIdx.x] = smid();
    a.trace[3 * blockIdx.x + 1] = gtimer();
  }
  __shared__ int s_gwork[NW][kGroupCols];
  __shared__ int s_gok[NW][kGroupCols];
  __shared__ double s_gpr[NW][kGroupCols];
  // dynamic shared memory: [double-double table x kTabCopies][single-double
  // table x kTab1Copies][per-warp scratch, deep_warp_doubles each]
  double2* s_tab_all = reinterpret_cast<double2*>(smem_raw);
  double* s_tab1_all = reinterpret_cast<double*>(s_tab_all + kExpTableSize * kTabCopies);
  if (VAR != kVarApprox) {
    for (int i = threadIdx.x; i < kExpTableSize * kTabCopies; i += blockDim.x)
      s_tab_all[i] = a.exp_tab[i / kTabCopies];
    for (int i = threadIdx.x; i < kExpTableSize * kTab1Copies; i += blockDim.x)
      s_tab1_all[i] = a.exp_tab[i / kTab1Copies].x;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const double2* s_tab = s_tab_all + (lane & (kTabCopies - 1));
  // opaque, so the lane's address stays in a register rather than being
  // rematerialised from %tid inside the Newton loop
  const unsigned tab1_addr = opaque_u32(smem_u32(s_tab1_all + (lane & (kTab1Copies - 1))));
  double* s_warp = s_tab1_all + kExpTableSize * kTab1Copies + (size_t)wib * deep_warp_doubles(NARROW, a.L);
  deep_worker<VAR, NARROW>(a, s_tab, tab1_addr, s_warp, s_gwork[wib], s_gok[wib], s_gpr[wib], lane);
#ifdef CVG_PHASE_CLOCKS
  __syncthreads();
  if (threadIdx.x < 8) atomicAdd(&g_phase[threadIdx.x], s_phase[threadIdx.x]);
#endif
  if (a.trace) {
    __syncthreads();
    if (threadIdx.x == 0) a.trace[3 * blockIdx.x + 2] = gtimer();
  }
}

// ---------------------------------------------------------------------------
// Thread-per-column deep kernel (large calls; CVG_DEEP_TPC):
// a warp claims 8 listed groups (32 column slots, lane = slot), every lane
// with a triggered column runs its column's levels in a loop (deep_level),
// storing each level row as it goes (coalesced across the warp's lanes when
// the groups are contiguous) and summing precip in k order (the
// reference's order); lanes of untriggered slots write the zeros.
// Calls with at least this many columns use it (convgpu.cu launch_kernels).
constexpr long long kTpcMinColumns = 320000;

// LPC lanes per column (1: one thread per column; 2, 4: a column's levels
// split round-robin over LPC lanes -- shorter claims, more columns per
// warp in flight).  ORD: precip summed in k order (the reference's order:
// strict, ApproxTranscendental); !ORD (relaxed path, tree_precip): each
// lane sums its levels in k order and the LPC partial sums are combined as
// a fixed-shape tree -- no per-round gathers (0.420 vs 0.434 ms at f02).
template <int VAR, int NW, int REGCAP, int LPC = 1, bool ORD = true>
__global__ void __maxnreg__(REGCAP) deep_tpc_kernel(DeepArgs a) {
  constexpr int kCols = 32 / LPC;              // columns per warp claim
  constexpr int kGroupsPerClaim = kCols / kGroupCols;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  if (a.trace && threadIdx.x == 0) {
    a.trace[3 * blockIdx.x] = smid();
    a.trace[3 * blockIdx.x + 1] = gtimer();
  }
  double2* s_tab_all = reinterpret_cast<double2*>(smem_raw);
  double* s_tab1_all = reinterpret_cast<double*>(s_tab_all + kExpTableSize * kTabCopies);
  if (VAR != kVarApprox) {
    for (int i = threadIdx.x; i < kExpTableSize * kTabCopies; i += blockDim.x)
      s_tab_all[i] = a.exp_tab[i / kTabCopies];
    for (int i = threadIdx.x; i < kExpTableSize * kTab1Copies; i += blockDim.x)
      s_tab1_all[i] = a.exp_tab[i / kTab1Copies].x;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int cs = lane / LPC, sub = lane % LPC;   // column slot, level phase
  const double2* s_tab = s_tab_all + (lane & (kTabCopies - 1));
  const unsigned tab1_addr = opaque_u32(smem_u32(s_tab1_all + (lane & (kTab1Copies - 1))));
  const long long G = *a.count;
  const int L = a.L;
  const unsigned lane_op = opaque_u32(lane);
  for (;;) {
    long long j = 0;
    if (lane == 0) j = (long long)atomicAdd(a.cursor + lane_op, (unsigned long long)kGroupsPerClaim);
    j = __shfl_sync(0xffffffffu, j, 0);
    if (j >= G) break;
    const long long x = j + cs / kGroupCols;
    const long long e = x < G ? a.groups[x] : -1;
    const int slot = cs & (kGroupCols - 1);
    const long long c = e >= 0 ? (e >> 4) * kGroupCols + slot : -1;
    const bool valid = c >= 0 && c < a.n;
    const bool trig = valid && ((e >> slot) & 1);
    double pr = 0.0;
    long long wsum = 0;
    bool ok = true;
    if (!ORD) {
      if (valid && !trig) {
        for (int k = sub; k < L; k += LPC) {
          a.tend_T[(long long)k * a.ld_out + c] = 0.0;
          a.tend_q[(long long)k * a.ld_out + c] = 0.0;
        }
      } else if (trig) {
        double* pT = a.tend_T + c;
        double* pQ = a.tend_q + c;
        const double sc = a.s[c];
        const double guess = add(24.0, mul(160.0, sc));
        const double rho = add(1.0, mul(kMC.c005, sc));
        const double e0 = deep_exp<VAR>(mul(kMC.c005, guess), s_tab);
        const double c0 = add(e0, mul(kMC.c001, guess));
        const bool col_far = guess < 512.0;
        const double* Tr = a.T + c;
        const double* qr = a.q + c;
        double Tn = 0.0, qn = 0.0;
        if (sub < L) {
          Tn = __ldg(Tr + (long long)sub * a.ld_in);
          qn = __ldg(qr + (long long)sub * a.ld_in);
        }
        for (int k = sub; k < L; k += LPC) {
          const double T = Tn, q = qn;
          if (k + LPC < L) {
            Tn = __ldg(Tr + (long long)(k + LPC) * a.ld_in);
            qn = __ldg(qr + (long long)(k + LPC) * a.ld_in);
          }
          double tT, tq, term;
          int w;
          if (!deep_level<VAR>(a, s_tab, tab1_addr, a.first_col + c, k, sc, rho, guess, e0, c0, col_far, T, q, tT,
                               tq, term, w))
            ok = false;
          pT[(long long)k * a.ld_out] = tT;
          pQ[(long long)k * a.ld_out] = tq;
          pr = add(pr, term);   // physics.cpp:161, k order (within the lane's levels)
          wsum += w;
        }
      }
      if (LPC > 1) {   // combine the column's lanes (fixed shape)
  #pragma unroll
        for (int o = LPC / 2; o > 0; o >>= 1) {
          pr = add(pr, __shfl_xor_sync(0xffffffffu, pr, o));
          wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
          ok = __shfl_xor_sync(0xffffffffu, (int)ok, o) && ok;
        }
      }
    } else {
      if (valid && !trig) {
        for (int k = sub; k < L; k += LPC) {
          a.tend_T[(long long)k * a.ld_out + c] = 0.0;
          a.tend_q[(long long)k * a.ld_out + c] = 0.0;
        }
      }
      // Levels in rounds: round r covers levels r LPC .. r LPC + LPC - 1, lane
      // sub takes level r LPC + sub.  Every lane of the warp runs the same
      // rounds, so after each one the column's LPC terms are gathered by warp
      // shuffles and added in k order (physics.cpp:161) -- the reference's
      // summation order for every LPC, every variant.
      double sc = 0.0, guess = 0.0, rho = 0.0, e0 = 0.0, c0 = 0.0;
      bool col_far = false;
      const double* Tr = a.T + (trig ? c : 0);
      const double* qr = a.q + (trig ? c : 0);
      double Tn = 0.0, qn = 0.0;
      if (trig) {
        sc = a.s[c];
        guess = add(24.0, mul(160.0, sc));
        rho = add(1.0, mul(kMC.c005, sc));
        e0 = deep_exp<VAR>(mul(kMC.c005, guess), s_tab);
        c0 = add(e0, mul(kMC.c001, guess));
        col_far = guess < 512.0;
        if (sub < L) {
          Tn = __ldg(Tr + (long long)sub * a.ld_in);
          qn = __ldg(qr + (long long)sub * a.ld_in);
        }
      }
      const int rounds = (L + LPC - 1) / LPC;
      for (int r = 0; r < rounds; ++r) {
        const int k = r * LPC + sub;
        double term = 0.0;
        if (trig && k < L) {
          const double T = Tn, q = qn;
          if (k + LPC < L) {
            Tn = __ldg(Tr + (long long)(k + LPC) * a.ld_in);
            qn = __ldg(qr + (long long)(k + LPC) * a.ld_in);
          }
          double tT, tq;
          int w;
          if (!deep_level<VAR>(a, s_tab, tab1_addr, a.first_col + c, k, sc, rho, guess, e0, c0, col_far, T, q, tT,
                               tq, term, w))
            ok = false;
          a.tend_T[(long long)k * a.ld_out + c] = tT;
          a.tend_q[(long long)k * a.ld_out + c] = tq;
          wsum += w;
        }
        if (LPC == 1) {
          pr = add(pr, term);
        } else {
  #pragma unroll
          for (int i2 = 0; i2 < LPC; ++i2) pr = add(pr, __shfl_sync(0xffffffffu, term, (lane & ~(LPC - 1)) + i2));
        }
      }
      if (LPC > 1) {   // the column's work count and success over its lanes
  #pragma unroll
        for (int o = LPC / 2; o > 0; o >>= 1) {
          wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
          ok = __shfl_xor_sync(0xffffffffu, (int)ok, o) && ok;
        }
      }
    }
    if (sub == 0 && valid) {
      if (!trig) {
        a.precip[c] = 0.0;
        a.work[c] = 0;
        a.exited[c] = 1;
      } else if (ok) {
        a.precip[c] = pr;
        a.work[c] = wsum;
        a.exited[c] = 0;
      }
    }
  }
  if (a.trace) {
    __syncthreads();
    if (threadIdx.x == 0) a.trace[3 * blockIdx.x + 2] = gtimer();
  }
}

// ---------------------------------------------------------------------------
// Feedback loop (validate.cpp:113-206): perturb_lsb, advance, check_finite
// and the RMS difference of two temperature fields.

// T[k][c] -> bits ^ 1 (perturb_lsb, validate.cpp:29-34); a non-finite value
// sets *bad (the reference throws ValidationError).
__global__ void perturb_lsb_kernel(double* T, long long ld, long long n, int L, unsigned* bad) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * L) return;
  const long long k = i / n, c = i - k * n;
  double* p = T + k * ld + c;
  const double x = *p;
  if (!is_finite(x)) atomicOr(bad, 1u);
  *p = __longlong_as_double(__double_as_longlong(x) ^ 1LL);
}

// T += tend_T, q += tend_q (advance, validate.cpp:127-136), one rounding
// each; a non-finite result sets *nonfinite (check_finite, :138-153).
__global__ void advance_kernel(double* T, double* q, long long ld, const double* __restrict__ tT,
                               const double* __restrict__ tq, long long ld_t, long long n, int L,
                               unsigned* nonfinite) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * L) return;
  const long long k = i / n, c = i - k * n;
  const double a = add(T[k * ld + c], tT[k * ld_t + c]);
  const double b = add(q[k * ld + c], tq[k * ld_t + c]);
  T[k * ld + c] = a;
  q[k * ld + c] = b;
  if (!is_finite(a) || !is_finite(b)) atomicOr(nonfinite, 1u);
}

// Sums of (Tm - Tb)^2 and (Tp - Tb)^2 over the [L][n] fields, in a fixed
// order (deterministic): block b reduces elements b, b + G, ... in a tree;
// rms_final_kernel adds the G partials in block order.
constexpr int kRmsThreads = 256;

__global__ void __launch_bounds__(kRmsThreads) rms_partial_kernel(const double* Tb, const double* Tm, const double* Tp,
                                                                  long long ld, long long n, int L,
                                                                  double* partials) {
  __shared__ double s0[kRmsThreads], s1[kRmsThreads];
  double a0 = 0.0, a1 = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n * L;
       i += (long long)gridDim.x * blockDim.x) {
    const long long k = i / n, c = i - k * n;
    const double b = Tb[k * ld + c];
    const double dm = sub(Tm[k * ld + c], b), dp = sub(Tp[k * ld + c], b);
    a0 = add(a0, mul(dm, dm));
    a1 = add(a1, mul(dp, dp));
  }
  s0[threadIdx.x] = a0;
  s1[threadIdx.x] = a1;
  __syncthreads();
  for (int o = kRmsThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      s0[threadIdx.x] = add(s0[threadIdx.x], s0[threadIdx.x + o]);
      s1[threadIdx.x] = add(s1[threadIdx.x], s1[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = s0[0];
    partials[2 * blockIdx.x + 1] = s1[0];
  }
}

__global__ void rms_final_kernel(const double* partials, int nblocks, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double a0 = 0.0, a1 = 0.0;
    for (int b = 0; b < nblocks; ++b) {
      a0 = add(a0, partials[2 * b]);
      a1 = add(a1, partials[2 * b + 1]);
    }
    out[0] = a0;
    out[1] = a1;
  }
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
  double t = guess;
  double e = deep_exp<VAR, 1>(mul(kMC.c005, t), s_tab);
  double resid = sub(add(e, mul(kMC.c001, t)), yy);
  for (int it = 0; it <= maxit; ++it) {
    if (fabs(resid) <= tol) { root[i] = t; iters[i] = it; return; }
    const double deriv = add(mul(kMC.c005, e), kMC.c001);
    t = sub(t, div_rn(resid, deriv));
    if (!is_finite(t)) { raise_failure(err, i, 0, kFailDiverged); return; }
    e = deep_exp<VAR, 1>(mul(kMC.c005, t), s_tab);
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
