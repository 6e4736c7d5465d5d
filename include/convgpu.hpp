// convgpu.hpp -- header-only C++ drop-in over the C ABI (convgpu.h).
//
// Mirrors the reference's column-batch entry points
//
//   std::vector<ColumnOutput> deep_convection(const Chunk&, const KernelOptions&)
//   std::vector<ColumnOutput> shallow_convection(const Chunk&, const KernelOptions&)
//       /root/reference/proj/src/core/physics.hpp:155-158
//
// for any Chunk / ColumnOutput / KernelOptions types shaped like the
// reference's (physics.hpp:32-73): Chunk{n_levels, first_col, cols},
// ColumnState{col_id, s, T, q}, ColumnOutput{tend_T, tend_q, precip,
// work_units, exited_early}, KernelOptions{variant, activity_threshold,
// newton_tol, newton_max_iter}.  With the reference headers on the include
// path a caller writes
//
//   cvg::Session gpu(0);
//   auto outs = gpu.deep_convection<convproxy::ColumnOutput, convproxy::KernelError>(chunk, opts);
//
// The AoS <-> level-major SoA marshalling happens on the host here; callers
// that already hold SoA buffers should use cvg_convect directly.  A numeric
// failure throws Error(message, column) -- the reference's KernelError
// signature (errors.hpp:26-36) -- naming the lowest failing column, exactly
// the column the serial driver would have thrown on; anything else throws
// std::runtime_error.  No CPU fallback: a missing device throws.
#pragma once

#include <chrono>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "convgpu.h"

namespace cvg {

namespace detail {

// AoS Chunk -> level-major SoA, one call through `call(in, opts, mask, out,
// stats)`, SoA -> std::vector<Output>.  marshal_ms: host time of the two
// conversions (hard part 6: reported beside the device time).
template <class Output, class Error, class Chunk, class Opts, class Call>
std::vector<Output> run_chunk(const Chunk& chunk, const Opts& opts, int mask, Call&& call, cvg_stats& stats,
                              double& marshal_ms) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  const long long n = static_cast<long long>(chunk.cols.size());
  const int L = chunk.n_levels;
  std::vector<double> s(n), T(static_cast<size_t>(n) * L), q(static_cast<size_t>(n) * L);
  for (long long c = 0; c < n; ++c) {
    const auto& col = chunk.cols[static_cast<size_t>(c)];
    s[c] = col.s;
    for (int k = 0; k < L; ++k) {
      T[static_cast<size_t>(k) * n + c] = col.T[static_cast<size_t>(k)];
      q[static_cast<size_t>(k) * n + c] = col.q[static_cast<size_t>(k)];
    }
  }
  const long long first = n > 0 ? static_cast<long long>(chunk.cols[0].col_id) : chunk.first_col;
  cvg_columns in{n, L, first, n, s.data(), T.data(), q.data(), 0};
  cvg_options o{static_cast<int>(opts.variant), opts.activity_threshold, opts.newton_tol, opts.newton_max_iter, 0};
  std::vector<double> tT(static_cast<size_t>(n) * L), tq(static_cast<size_t>(n) * L), pr(n);
  std::vector<long long> wk(n);
  std::vector<uint8_t> ex(n);
  cvg_outputs out{tT.data(), tq.data(), pr.data(), wk.data(), ex.data(), n, 0};
  const auto t1 = clk::now();
  const cvg_status st = call(&in, &o, mask, &out, &stats);
  if (st == CVG_ERR_NUMERIC) throw Error(cvg_last_error(), stats.failing_column);
  if (st != CVG_OK) throw std::runtime_error(cvg_last_error());
  const auto t2 = clk::now();
  std::vector<Output> outs(static_cast<size_t>(n));
  for (long long c = 0; c < n; ++c) {
    Output& r = outs[static_cast<size_t>(c)];
    r.tend_T.resize(static_cast<size_t>(L));
    r.tend_q.resize(static_cast<size_t>(L));
    for (int k = 0; k < L; ++k) {
      r.tend_T[static_cast<size_t>(k)] = tT[static_cast<size_t>(k) * n + c];
      r.tend_q[static_cast<size_t>(k)] = tq[static_cast<size_t>(k) * n + c];
    }
    r.precip = pr[c];
    r.work_units = wk[c];
    r.exited_early = ex[c] != 0;
  }
  marshal_ms = std::chrono::duration<double, std::milli>((t1 - t0) + (clk::now() - t2)).count();
  return outs;
}

}  // namespace detail

class Session {
 public:
  explicit Session(int device = 0) {
    if (cvg_context_create(device, &ctx_) != CVG_OK) throw std::runtime_error(cvg_last_error());
  }
  ~Session() { cvg_context_free(ctx_); }
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;

  cvg_context* handle() const { return ctx_; }
  const cvg_stats& last_stats() const { return stats_; }
  // host time of the last call's AoS <-> SoA conversions
  double last_marshal_ms() const { return marshal_ms_; }

  template <class Output, class Error = std::runtime_error, class Chunk, class Opts>
  std::vector<Output> deep_convection(const Chunk& chunk, const Opts& opts) {
    return run<Output, Error>(chunk, opts, CVG_DEEP);
  }

  template <class Output, class Error = std::runtime_error, class Chunk, class Opts>
  std::vector<Output> shallow_convection(const Chunk& chunk, const Opts& opts) {
    return run<Output, Error>(chunk, opts, CVG_SHALLOW);
  }

 private:
  template <class Output, class Error, class Chunk, class Opts>
  std::vector<Output> run(const Chunk& chunk, const Opts& opts, int mask) {
    return detail::run_chunk<Output, Error>(
        chunk, opts, mask,
        [&](const cvg_columns* in, const cvg_options* o, int m, const cvg_outputs* out, cvg_stats* st) {
          return cvg_convect(ctx_, in, o, m, m == CVG_DEEP ? out : nullptr, m == CVG_SHALLOW ? out : nullptr, st);
        },
        stats_, marshal_ms_);
  }

  cvg_context* ctx_ = nullptr;
  cvg_stats stats_{};
  double marshal_ms_ = 0.0;
};

// The same entry points over several devices (cvg_multi): the chunk is split
// into contiguous column ranges balanced by estimated cost and computed on
// every device concurrently -- HeteroEngine::step (hetero.cpp:252-466) over
// G devices, with the same outputs as one Session call.
class MultiSession {
 public:
  explicit MultiSession(const std::vector<int>& devices) {
    if (cvg_multi_create(devices.data(), static_cast<int>(devices.size()), &m_) != CVG_OK)
      throw std::runtime_error(cvg_last_error());
    bounds_.assign(devices.size() + 1, 0);
  }
  ~MultiSession() { cvg_multi_free(m_); }
  MultiSession(const MultiSession&) = delete;
  MultiSession& operator=(const MultiSession&) = delete;

  cvg_multi* handle() const { return m_; }
  const cvg_stats& last_stats() const { return stats_; }
  double last_marshal_ms() const { return marshal_ms_; }
  // the last call's range offsets (devices + 1 entries)
  const std::vector<long long>& last_bounds() const { return bounds_; }

  template <class Output, class Error = std::runtime_error, class Chunk, class Opts>
  std::vector<Output> deep_convection(const Chunk& chunk, const Opts& opts) {
    return run<Output, Error>(chunk, opts, CVG_DEEP);
  }

  template <class Output, class Error = std::runtime_error, class Chunk, class Opts>
  std::vector<Output> shallow_convection(const Chunk& chunk, const Opts& opts) {
    return run<Output, Error>(chunk, opts, CVG_SHALLOW);
  }

 private:
  template <class Output, class Error, class Chunk, class Opts>
  std::vector<Output> run(const Chunk& chunk, const Opts& opts, int mask) {
    return detail::run_chunk<Output, Error>(
        chunk, opts, mask,
        [&](const cvg_columns* in, const cvg_options* o, int m, const cvg_outputs* out, cvg_stats* st) {
          return cvg_multi_convect(m_, in, o, m, m == CVG_DEEP ? out : nullptr, m == CVG_SHALLOW ? out : nullptr, st,
                                   bounds_.data());
        },
        stats_, marshal_ms_);
  }

  cvg_multi* m_ = nullptr;
  cvg_stats stats_{};
  double marshal_ms_ = 0.0;
  std::vector<long long> bounds_;
};

}  // namespace cvg
