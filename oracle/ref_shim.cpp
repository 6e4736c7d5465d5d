// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim, written for this repo, over the UNMODIFIED reference sources
// /root/reference/proj/src/core/{physics,sched,validate,hetero}.cpp, which oracle/Makefile
// compiles in place (read-only) into oracle/_ref/libconvref.so with the
// reference's own flags (-std=c++20 -O3 -DNDEBUG -ffp-contract=off,
// proj/CMakeLists.txt:12-15).  No reference source is copied into this repo.
//
// It marshals the level-major SoA layout into the reference's AoS Chunk
// (physics.hpp:32-43), calls the reference entry points, and unmarshals.
// Used to (1) pin the C restatement oracle/convproxy_oracle.c bit-for-bit,
// (2) generate tests/golden/ fixtures, and (3) time the reference's own
// run_parallel (sched.hpp:73-74) as bench.py's CPU baseline.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "bench.hpp"
#include "errors.hpp"
#include "hetero.hpp"
#include "physics.hpp"
#include "sched.hpp"
#include "validate.hpp"

using namespace convproxy;

namespace {

KernelOptions make_opts(int variant, double thr, double tol, int maxit) {
  KernelOptions o;
  o.variant = variant == 1   ? Variant::StrengthReduced
              : variant == 2 ? Variant::ApproxTranscendental
                             : Variant::Exact;
  o.activity_threshold = thr;
  o.newton_tol = tol;
  o.newton_max_iter = maxit;
  return o;
}

Chunk to_chunk(long long n, int L, long long ld, long long first_col,
               const double* s, const double* T, const double* q) {
  Chunk ch;
  ch.n_levels = L;
  ch.first_col = first_col;
  ch.cols.resize(static_cast<size_t>(n));
  for (long long c = 0; c < n; ++c) {
    ColumnState& col = ch.cols[static_cast<size_t>(c)];
    col.col_id = first_col + c;
    col.s = s[c];
    col.T.resize(static_cast<size_t>(L));
    col.q.resize(static_cast<size_t>(L));
    for (int k = 0; k < L; ++k) {
      col.T[static_cast<size_t>(k)] = T[k * ld + c];
      col.q[static_cast<size_t>(k)] = q[k * ld + c];
    }
  }
  return ch;
}

void from_outputs(const std::vector<ColumnOutput>& outs, int L, long long ld,
                  double* tend_T, double* tend_q, double* precip,
                  long long* work, unsigned char* exited) {
  for (size_t c = 0; c < outs.size(); ++c) {
    const ColumnOutput& o = outs[c];
    for (int k = 0; k < L; ++k) {
      tend_T[k * ld + static_cast<long long>(c)] = o.tend_T[static_cast<size_t>(k)];
      tend_q[k * ld + static_cast<long long>(c)] = o.tend_q[static_cast<size_t>(k)];
    }
    precip[c] = o.precip;
    work[c] = o.work_units;
    exited[c] = o.exited_early ? 1 : 0;
  }
}

}  // namespace

extern "C" {

// 0 ok, 3 KernelError (fail_col set), 1 other failure.
int ref_convection(int kernel, long long n, int L, long long ld,
                   long long first_col, const double* s, const double* T,
                   const double* q, int variant, double thr, double tol,
                   int maxit, double* tend_T, double* tend_q, double* precip,
                   long long* work, unsigned char* exited,
                   long long* fail_col) {
  try {
    const Chunk ch = to_chunk(n, L, ld, first_col, s, T, q);
    const KernelOptions o = make_opts(variant, thr, tol, maxit);
    const std::vector<ColumnOutput> outs =
        kernel == 0 ? deep_convection(ch, o) : shallow_convection(ch, o);
    from_outputs(outs, L, ld, tend_T, tend_q, precip, work, exited);
    return 0;
  } catch (const KernelError& e) {
    if (fail_col) *fail_col = e.column();
    return 3;
  } catch (...) {
    return 1;
  }
}

int ref_ientropy_solve(double y, double guess, int variant, double tol,
                       int maxit, double* root, int* iterations) {
  try {
    const IentropyResult r =
        ientropy_solve(y, guess, make_opts(variant, 0.5, tol, maxit));
    *root = r.root;
    *iterations = r.iterations;
    return 0;
  } catch (const KernelError&) {
    return 3;
  } catch (...) {
    return 1;
  }
}

double ref_approx_exp(double x) { return approx_exp(x); }

void ref_make_grid(long long n, int L, double band, unsigned long long seed,
                   double* s, double* T, double* q) {
  GridSpec spec;
  spec.n_columns = n;
  spec.n_levels = L;
  spec.tropics_band = band;
  spec.seed = seed;
  const Chunk g = make_grid(spec);
  for (long long c = 0; c < n; ++c) {
    const ColumnState& col = g.cols[static_cast<size_t>(c)];
    s[c] = col.s;
    for (int k = 0; k < L; ++k) {
      T[k * n + c] = col.T[static_cast<size_t>(k)];
      q[k * n + c] = col.q[static_cast<size_t>(k)];
    }
  }
}

// ---- CPU baseline timing through the reference's own scheduler ----------

void* ref_chunk_create(long long n, int L, long long ld, long long first_col,
                       const double* s, const double* T, const double* q) {
  try {
    return new Chunk(to_chunk(n, L, ld, first_col, s, T, q));
  } catch (...) {
    return nullptr;
  }
}

void ref_chunk_free(void* h) { delete static_cast<Chunk*>(h); }

// Times run_parallel(chunk, deep_column|shallow_column, opts,
// {strategy, omp_chunk, n_threads}) (sched.cpp:78-208).  strategy:
// 0 StaticBlock, 1 StaticCyclic, 2 Dynamic, 3 TaskPerColumn.
// Returns 0 ok / 3 KernelError / 1 other; *wall_s is the reference's own
// RunMetrics::wall_s.  Optional SoA outputs (any may be null -> skipped).
int ref_run_parallel(void* h, int kernel, int variant, double thr, double tol,
                     int maxit, int n_threads, int strategy, int omp_chunk,
                     double* wall_s, double* tend_T, double* tend_q,
                     double* precip, long long* work, unsigned char* exited) {
  try {
    const Chunk& ch = *static_cast<Chunk*>(h);
    ScheduleSpec spec;
    spec.strategy = static_cast<Strategy>(strategy);
    spec.omp_chunk_size = omp_chunk;
    spec.n_threads = n_threads;
    const KernelFn fn = kernel == 0 ? &deep_column : &shallow_column;
    const RunResult r =
        run_parallel(ch, fn, make_opts(variant, thr, tol, maxit), spec);
    if (wall_s) *wall_s = r.metrics.wall_s;
    if (tend_T && tend_q && precip && work && exited) {
      from_outputs(r.outputs, ch.n_levels,
                   static_cast<long long>(ch.cols.size()), tend_T, tend_q,
                   precip, work, exited);
    }
    return 0;
  } catch (const KernelError&) {
    return 3;
  } catch (...) {
    return 1;
  }
}

// ---- staging byte accounting (hetero.cpp:178-201, :268-312, :336-374) -----
//
// The reference's device staging packs T, q, s (+ the 4-double option block
// "env" unless scalars are resident) into one 8-byte-aligned payload, and the
// outputs tend_T, tend_q, precip, work_units, exited into another; bytes_in /
// bytes_out are the payload sizes (HeteroMetrics, hetero.hpp:120-131).  This
// reproduces them with the reference's own pack() for nd device columns.
int ref_packed_bytes(long long nd, int L, int send_scalars, long long* bytes_in, long long* bytes_out) {
  try {
    std::vector<double> tl(static_cast<size_t>(nd * L)), ql(tl.size()), sl(static_cast<size_t>(nd));
    double env[4] = {0.5, 1e-12, 100.0, 0.0};
    std::vector<NamedArray> in = {
        {"T", tl.data(), tl.size() * sizeof(double)},
        {"q", ql.data(), ql.size() * sizeof(double)},
        {"s", sl.data(), sl.size() * sizeof(double)},
    };
    if (send_scalars) in.push_back({"env", env, sizeof(env)});
    *bytes_in = static_cast<long long>(pack(in).payload.size());
    std::vector<double> pr(static_cast<size_t>(nd));
    std::vector<long long> wu(static_cast<size_t>(nd));
    std::vector<std::uint8_t> ex(static_cast<size_t>(nd));
    *bytes_out = static_cast<long long>(pack({{"tend_T", tl.data(), tl.size() * sizeof(double)},
                                              {"tend_q", ql.data(), ql.size() * sizeof(double)},
                                              {"precip", pr.data(), pr.size() * sizeof(double)},
                                              {"work_units", wu.data(), wu.size() * sizeof(long long)},
                                              {"exited", ex.data(), ex.size()}})
                                             .payload.size());
    return 0;
  } catch (...) {
    return 1;
  }
}

// ---- BenchRecord CSV (bench.cpp:454-525) ------------------------------------
//
// Parses a records CSV with the reference's own records_from_csv and writes
// it back with records_to_csv: 0 ok (*n_records set, out receives the
// re-serialised CSV when it fits), 2 ConfigError (message in out), 1 other.
int ref_records_roundtrip(const char* csv, int* n_records, char* out, int out_len) {
  try {
    const std::vector<BenchRecord> recs = records_from_csv(csv);
    *n_records = static_cast<int>(recs.size());
    const std::string s = records_to_csv(recs);
    if (out && out_len > 0) {
      std::strncpy(out, s.c_str(), static_cast<size_t>(out_len - 1));
      out[out_len - 1] = 0;
    }
    return 0;
  } catch (const ConfigError& e) {
    if (out && out_len > 0) {
      std::strncpy(out, e.what(), static_cast<size_t>(out_len - 1));
      out[out_len - 1] = 0;
    }
    return 2;
  } catch (...) {
    return 1;
  }
}

// ---- error_growth (validate.cpp:168-206) -----------------------------------
//
// Three legs from the same grid for `timesteps` steps of T += tend_T,
// q += tend_q with kernel deep_column (0) or shallow_column (1): baseline
// (variant vb), modified (variant vm), perturbed (initial T one ulp off,
// variant vb).  Both paths serial StaticBlock, as acceptance.cpp:570-573.
// Returns 0 ok, 3 KernelError, 4 ValidationError (*fail_step set), 1 other.
int ref_error_growth(int kernel, long long n, int L, const double* s, const double* T, const double* q,
                     int vb, int vm, double thr, double tol, int maxit, int timesteps, double* rms_mod,
                     double* rms_pert, int* envelope_ok, double* worst_ratio, int* fail_step) {
  try {
    const Chunk ch = to_chunk(n, L, n, 0, s, T, q);
    SimPath base;
    base.opts = make_opts(vb, thr, tol, maxit);
    base.sched.strategy = Strategy::StaticBlock;
    base.sched.n_threads = 1;
    SimPath mod = base;
    mod.opts = make_opts(vm, thr, tol, maxit);
    const KernelFn fn = kernel == 0 ? &deep_column : &shallow_column;
    const ErrorGrowthSeries r = error_growth(ch, fn, base, mod, timesteps);
    for (size_t i = 0; i < r.rms_mod.size(); ++i) {
      rms_mod[i] = r.rms_mod[i];
      rms_pert[i] = r.rms_pert[i];
    }
    *envelope_ok = r.envelope_ok ? 1 : 0;
    *worst_ratio = r.worst_ratio;
    return 0;
  } catch (const KernelError&) {
    return 3;
  } catch (const ValidationError& e) {
    if (fail_step) *fail_step = e.timestep();
    return 4;
  } catch (...) {
    return 1;
  }
}

}  // extern "C"
