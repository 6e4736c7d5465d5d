// test_dropin.cpp -- the drop-in, exercised the way the reference's own tests
// exercise its kernels (proj/tests/test_physics.cpp), with the reference's
// own types and its own CPU implementation as the comparison:
// convproxy::deep_convection / shallow_convection from oracle/_ref (the
// reference's physics.cpp compiled unmodified) versus cvg::Session (the
// B200 path through include/convgpu.hpp -> convgpu.h).
//
// Built in the build container (needs /root/reference headers) by
// tests/cpp/Makefile; run on the GPU box by tests/test_dropin_gpu.py.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "convgpu.hpp"
#include "errors.hpp"
#include "physics.hpp"

using namespace convproxy;

static int g_fail = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
      ++g_fail;                                                       \
    }                                                                 \
  } while (0)

static bool close_fields(const ColumnOutput& a, const ColumnOutput& b) {
  auto ok = [](double x, double y) { return std::fabs(x - y) <= std::fmax(1e-10 * std::fabs(y), 1e-14); };
  if (a.tend_T.size() != b.tend_T.size() || a.exited_early != b.exited_early) return false;
  for (size_t k = 0; k < a.tend_T.size(); ++k)
    if (!ok(a.tend_T[k], b.tend_T[k]) || !ok(a.tend_q[k], b.tend_q[k])) return false;
  return ok(a.precip, b.precip);
}

static bool bitwise(const ColumnOutput& a, const ColumnOutput& b) {
  auto eq = [](double x, double y) { return std::memcmp(&x, &y, 8) == 0; };
  for (size_t k = 0; k < a.tend_T.size(); ++k)
    if (!eq(a.tend_T[k], b.tend_T[k]) || !eq(a.tend_q[k], b.tend_q[k])) return false;
  return eq(a.precip, b.precip) && a.work_units == b.work_units && a.exited_early == b.exited_early;
}

int main() {
  cvg::Session gpu(0);
  KernelOptions exact;

  {  // test_physics.cpp:248-262 -- deep kernel vs reference (tolerance rule)
    GridSpec spec;
    spec.n_columns = 64;
    spec.seed = 7;
    const Chunk grid = make_grid(spec);
    const auto want = deep_convection(grid, exact);
    const auto got = gpu.deep_convection<ColumnOutput, KernelError>(grid, exact);
    int active = 0;
    for (size_t i = 0; i < want.size(); ++i) {
      CHECK(close_fields(got[i], want[i]));
      CHECK(got[i].work_units == want[i].work_units);
      if (!got[i].exited_early) ++active;
    }
    CHECK(active > 10);
  }
  {  // test_physics.cpp:227-246 -- inactive columns: zeros, work 0
    GridSpec spec;
    spec.n_columns = 32;
    spec.tropics_band = 0.0;
    for (const ColumnOutput& o : gpu.deep_convection<ColumnOutput, KernelError>(make_grid(spec), exact)) {
      CHECK(o.exited_early);
      CHECK(o.work_units == 0);
    }
  }
  {  // test_physics.cpp:380-390 + 392-415 -- shallow vs reference, exits spread
    GridSpec spec;
    spec.n_columns = 256;
    spec.seed = 3;
    const Chunk grid = make_grid(spec);
    const auto want = shallow_convection(grid, exact);
    const auto got = gpu.shallow_convection<ColumnOutput, KernelError>(grid, exact);
    int by_phase[5] = {0, 0, 0, 0, 0};
    for (size_t i = 0; i < want.size(); ++i) {
      CHECK(close_fields(got[i], want[i]));
      CHECK(got[i].work_units == want[i].work_units);
      by_phase[got[i].exited_early ? got[i].work_units / 30 - 1 : 4]++;
    }
    CHECK(by_phase[0] > 0 && by_phase[1] > 0 && by_phase[4] > 0);
  }
  {  // approx-exp variant: Newton path is pure IEEE -> work and precip bitwise
    KernelOptions approx;
    approx.variant = Variant::ApproxTranscendental;
    GridSpec spec;
    spec.n_columns = 20000;
    spec.seed = 11;
    const Chunk grid = make_grid(spec);
    const auto want = deep_convection(grid, approx);
    const auto got = gpu.deep_convection<ColumnOutput, KernelError>(grid, approx);
    long long bad = 0;
    for (size_t i = 0; i < want.size(); ++i) {
      double a = got[i].precip, b = want[i].precip;
      if (got[i].work_units != want[i].work_units || std::memcmp(&a, &b, 8) != 0 || !close_fields(got[i], want[i]))
        ++bad;
    }
    CHECK(bad == 0);
  }
  {  // test_physics.cpp:417-427 -- strength-reduced bit-identical when q == 0
    GridSpec spec;
    spec.n_columns = 16;
    spec.tropics_band = 1.0;
    Chunk grid = make_grid(spec);
    for (auto& c : grid.cols)
      for (double& q : c.q) q = 0.0;
    KernelOptions reduced;
    reduced.variant = Variant::StrengthReduced;
    const auto a = gpu.deep_convection<ColumnOutput, KernelError>(grid, exact);
    const auto b = gpu.deep_convection<ColumnOutput, KernelError>(grid, reduced);
    for (size_t i = 0; i < a.size(); ++i) CHECK(bitwise(a[i], b[i]));
  }
  {  // test_physics.cpp:488-501 -- KernelError carries column 5
    GridSpec spec;
    spec.n_columns = 8;
    spec.tropics_band = 1.0;
    Chunk grid = make_grid(spec);
    grid.cols[5].T[3] = std::nan("");
    bool thrown = false;
    try {
      gpu.deep_convection<ColumnOutput, KernelError>(grid, exact);
    } catch (const KernelError& e) {
      thrown = true;
      CHECK(e.column() == 5);
    }
    CHECK(thrown);
  }
  {  // the multi-device engine (HeteroEngine::step over G devices): a 4-way
     // split -- one GPU listed four times on a one-GPU box -- equals the
     // single-device call bit for bit and the reference within its rule
    GridSpec spec;
    spec.n_columns = 50000;
    spec.seed = 21;
    const Chunk grid = make_grid(spec);
    cvg::MultiSession multi({0, 0, 0, 0});
    const auto want = deep_convection(grid, exact);
    const auto one = gpu.deep_convection<ColumnOutput, KernelError>(grid, exact);
    const auto four = multi.deep_convection<ColumnOutput, KernelError>(grid, exact);
    long long differ = 0, off = 0;
    for (size_t i = 0; i < want.size(); ++i) {
      if (!bitwise(one[i], four[i])) ++differ;
      if (!close_fields(four[i], want[i]) || four[i].work_units != want[i].work_units) ++off;
    }
    CHECK(differ == 0);
    CHECK(off == 0);
    const auto& b = multi.last_bounds();
    CHECK(b.size() == 5 && b.front() == 0 && b.back() == 50000);
    for (size_t i = 1; i + 1 < b.size(); ++i) CHECK(b[i] % 32 == 0 && b[i] > b[i - 1]);
    CHECK(multi.last_stats().n_triggered == gpu.last_stats().n_triggered);
    CHECK(multi.last_marshal_ms() > 0.0);
    std::printf("multi: bounds %lld %lld %lld %lld %lld, marshal %.2f ms, device %.2f ms\n", b[0], b[1], b[2], b[3],
                b[4], multi.last_marshal_ms(), multi.last_stats().device_ms);
    Chunk bad = grid;   // failures in two ranges: the lowest column is reported
    for (auto& c : bad.cols) c.s = 0.9;
    bad.cols[41000].T[2] = std::nan("");
    bad.cols[9000].T[7] = std::nan("");
    bool thrown = false;
    try {
      multi.deep_convection<ColumnOutput, KernelError>(bad, exact);
    } catch (const KernelError& e) {
      thrown = true;
      CHECK(e.column() == 9000);
    }
    CHECK(thrown);
  }
  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "PASSED", g_fail);
  return g_fail ? 1 : 0;
}
