// Design probe: Newton-update throughput and exactness of the device math
// options in colmath.cuh (exp / division), measured on B200.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1711_00289_b200/csrc/colmath.cuh"

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

using namespace cvg;

template <int V> __device__ __forceinline__ double expv(double x, const double2* tab) {
  if (V == 0) return exp(x);
  if (V == 3) return approx_exp_ref(x);
  return exp_tang(x, tab);
}
template <int V> __device__ __forceinline__ double divv(double a, double b) {
  if (V == 0 || V == 1) return __ddiv_rn(a, b);
  return div_rn(a, b);
}

template <int V>
__global__ void __launch_bounds__(256) newton_k(const double* ys, const double* gs, int nsolve,
                                                double tol, int maxit, double* roots, int* iters,
                                                const double2* gtab) {
  __shared__ double2 tab[128];
  for (int i = threadIdx.x; i < 128; i += blockDim.x) tab[i] = gtab[i];
  __syncthreads();
  const long long nthr = (long long)gridDim.x * blockDim.x;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (int s = 0; s < nsolve; ++s) {
    const long long idx = s * nthr + tid;
    const double y = ys[idx], guess = gs[idx];
    double t = guess;
    double e = expv<V>(mul(0.05, t), tab);
    double resid = sub(add(e, mul(0.01, t)), y);
    int it = 0;
    while (!(fabs(resid) <= tol)) {
      if (it > maxit) { it = -1; break; }
      const double deriv = add(mul(0.05, e), 0.01);
      t = sub(t, divv<V>(resid, deriv));
      e = expv<V>(mul(0.05, t), tab);
      resid = sub(add(e, mul(0.01, t)), y);
      ++it;
    }
    roots[idx] = t;
    iters[idx] = it;
  }
}

__global__ void exp_k(const double* x, double* o_tang, double* o_cuda, double* o_apx, int n,
                      const double2* tab) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    o_tang[i] = exp_tang(x[i], tab);
    o_cuda[i] = exp(x[i]);
    o_apx[i] = approx_exp_ref(x[i]);
  }
}
__global__ void div_k(const double* a, const double* b, double* o, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = div_rn(a[i], b[i]);
}

static uint64_t sm64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static double u01(uint64_t c) { return (double)(sm64(c) >> 11) * 0x1.0p-53; }

static double host_approx_exp(double x) {
  const double kLn2Hi = 6.93147180369123816490e-01, kLn2Lo = 1.90821492927058770002e-10,
               kInvLn2 = 1.44269504088896338700e+00;
  const double kd = std::nearbyint(x * kInvLn2);
  const int k = (int)kd;
  const double r = (x - kd * kLn2Hi) - kd * kLn2Lo;
  double p = 1.0 / 479001600.0;
  p = p * r + 1.0 / 39916800.0; p = p * r + 1.0 / 3628800.0; p = p * r + 1.0 / 362880.0;
  p = p * r + 1.0 / 40320.0; p = p * r + 1.0 / 5040.0; p = p * r + 1.0 / 720.0;
  p = p * r + 1.0 / 120.0; p = p * r + 1.0 / 24.0; p = p * r + 1.0 / 6.0;
  p = p * r + 0.5; p = p * r + 1.0; p = p * r + 1.0;
  return std::ldexp(p, k);
}

static void host_newton(double y, double guess, bool apx, double* root, int* iters) {
  double t = guess;
  double e = apx ? host_approx_exp(0.05 * t) : std::exp(0.05 * t);
  double resid = e + 0.01 * t - y;
  int it = 0;
  while (!(std::fabs(resid) <= 1e-12)) {
    if (it > 100) { it = -1; break; }
    const double deriv = 0.05 * e + 0.01;
    t -= resid / deriv;
    e = apx ? host_approx_exp(0.05 * t) : std::exp(0.05 * t);
    resid = e + 0.01 * t - y;
    ++it;
  }
  *root = t; *iters = it;
}

int main() {
  // 2^(j/128) double-double table from long double
  std::vector<double2> tab(128);
  for (int j = 0; j < 128; ++j) {
    long double v = exp2l((long double)j / 128.0L);
    double hi = (double)v;
    double lo = (double)(v - (long double)hi);
    tab[j] = make_double2(hi, lo);
  }
  double2* dtab; CK(cudaMalloc(&dtab, 128 * sizeof(double2)));
  CK(cudaMemcpy(dtab, tab.data(), 128 * sizeof(double2), cudaMemcpyHostToDevice));

  // ---- exp accuracy vs glibc
  {
    const int n = 1 << 22;
    std::vector<double> x(n);
    for (int i = 0; i < n; ++i) x[i] = -1.25 + 10.75 * u01(i);
    double *dx, *a, *b, *c; CK(cudaMalloc(&dx, n * 8)); CK(cudaMalloc(&a, n * 8));
    CK(cudaMalloc(&b, n * 8)); CK(cudaMalloc(&c, n * 8));
    CK(cudaMemcpy(dx, x.data(), n * 8, cudaMemcpyHostToDevice));
    exp_k<<<(n + 255) / 256, 256>>>(dx, a, b, c, n, dtab);
    CK(cudaDeviceSynchronize());
    std::vector<double> ha(n), hb(n), hc(n);
    CK(cudaMemcpy(ha.data(), a, n * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hb.data(), b, n * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hc.data(), c, n * 8, cudaMemcpyDeviceToHost));
    long long dt = 0, dc = 0, da = 0, dtc = 0;
    for (int i = 0; i < n; ++i) {
      double g = std::exp(x[i]);
      if (memcmp(&g, &ha[i], 8)) ++dt;
      if (memcmp(&g, &hb[i], 8)) ++dc;
      double ap = host_approx_exp(x[i]);
      if (memcmp(&ap, &hc[i], 8)) ++da;
      if (memcmp(&ha[i], &hb[i], 8)) ++dtc;
    }
    printf("{\"probe\": \"exp_bits_vs_glibc\", \"n\": %d, \"tang_diff\": %lld, \"cuda_diff\": %lld, \"approx_ref_diff_vs_host_approx\": %lld, \"tang_vs_cuda\": %lld}\n",
           n, dt, dc, da, dtc);
    // division exactness
    std::vector<double> A(n), B(n);
    for (int i = 0; i < n; ++i) {
      A[i] = (u01(3 * i) - 0.5) * std::ldexp(1.0, (int)(u01(3 * i + 1) * 200) - 100);
      B[i] = 0.07 + 1000.0 * u01(3 * i + 2);
    }
    CK(cudaMemcpy(dx, A.data(), n * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(a, B.data(), n * 8, cudaMemcpyHostToDevice));
    div_k<<<(n + 255) / 256, 256>>>(dx, a, b, n);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(hb.data(), b, n * 8, cudaMemcpyDeviceToHost));
    long long dd = 0;
    for (int i = 0; i < n; ++i) { double g = A[i] / B[i]; if (memcmp(&g, &hb[i], 8)) ++dd; }
    printf("{\"probe\": \"div_rn_bits_vs_host\", \"n\": %d, \"diff\": %lld}\n", n, dd);
  }

  // ---- Newton throughput
  const int blocks = 148 * 8, threads = 256, nsolve = 64;
  const long long nthr = (long long)blocks * threads, N = nthr * nsolve;
  std::vector<double> ys(N), gs(N);
  for (long long i = 0; i < N; ++i) {
    const long long tid = i % nthr, s = i / nthr;
    const long long warp = tid / 32;
    ys[i] = 1.2 + 0.15 * u01(2 * i);
    gs[i] = 104.0 + 80.0 * u01(1000003 * s + warp);  // warp-uniform guess
  }
  double *dys, *dgs, *droots; int* dit;
  CK(cudaMalloc(&dys, N * 8)); CK(cudaMalloc(&dgs, N * 8)); CK(cudaMalloc(&droots, N * 8));
  CK(cudaMalloc(&dit, N * 4));
  CK(cudaMemcpy(dys, ys.data(), N * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dgs, gs.data(), N * 8, cudaMemcpyHostToDevice));
  std::vector<double> roots(N); std::vector<int> its(N);
  // host references on a subset
  const long long NCHK = 200000;
  std::vector<double> r_ex(NCHK), r_ap(NCHK); std::vector<int> i_ex(NCHK), i_ap(NCHK);
  for (long long i = 0; i < NCHK; ++i) {
    host_newton(ys[i], gs[i], false, &r_ex[i], &i_ex[i]);
    host_newton(ys[i], gs[i], true, &r_ap[i], &i_ap[i]);
  }
  auto run = [&](int V, const char* name, auto kern) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w = 0; w < 2; ++w) kern<<<blocks, threads>>>(dys, dgs, nsolve, 1e-12, 100, droots, dit, dtab);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      kern<<<blocks, threads>>>(dys, dgs, nsolve, 1e-12, 100, droots, dit, dtab);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    CK(cudaMemcpy(roots.data(), droots, N * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(its.data(), dit, N * 4, cudaMemcpyDeviceToHost));
    long long upd = 0; for (long long i = 0; i < N; ++i) upd += its[i];
    const bool apx = (V == 3);
    long long it_diff = 0, root_bits = 0; double max_rel = 0;
    for (long long i = 0; i < NCHK; ++i) {
      const double rr = apx ? r_ap[i] : r_ex[i]; const int ii = apx ? i_ap[i] : i_ex[i];
      if (ii != its[i]) ++it_diff;
      if (memcmp(&rr, &roots[i], 8)) ++root_bits;
      double rel = std::fabs(rr - roots[i]) / std::fabs(rr); if (rel > max_rel) max_rel = rel;
    }
    printf("{\"probe\": \"newton_%s\", \"ms\": %.4f, \"updates\": %lld, \"Gupd_per_s\": %.2f, \"mean_iters\": %.3f, \"chk_iter_diff\": %lld, \"chk_root_bitdiff\": %lld, \"chk_root_maxrel\": %.3g}\n",
           name, best, upd, upd / (best * 1e-3) / 1e9, (double)upd / N, it_diff, root_bits, max_rel);
  };
  run(0, "cudaexp_ieeediv", newton_k<0>);
  run(1, "tang_ieeediv", newton_k<1>);
  run(2, "tang_divrn", newton_k<2>);
  run(3, "approxref_divrn", newton_k<3>);
  return 0;
}
