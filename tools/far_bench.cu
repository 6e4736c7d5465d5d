// Design probe: the two-solve Newton loop with and without the FP32 far
// phase (colmath.cuh newton_far32_step) -- throughput versus warps per SM,
// and per-solve update counts / roots of the two variants compared (counts
// may differ only where a residual lands within rounding noise of tol).
// Inputs as tools/loop_bench.cu: y ~ U(1.2, 1.35), guess 24 + 160 s,
// s ~ U(0.5, 1) shared by the warp.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1711_00289_b200/csrc/colmath.cuh"
#include "../paper_1711_00289_b200/csrc/bulkcopy.cuh"

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

using namespace cvg;

__device__ __forceinline__ double u01(unsigned long long x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return (double)(x >> 11) * 0x1.0p-53;
}

template <bool FAR>
__global__ void loop_k(const double2* gtab, int cols, double tol, unsigned long long* iters_out, double* sink,
                       int* counts, double* roots) {
  extern __shared__ double s_tab1[];
  for (int i = threadIdx.x; i < kExpTableSize * kTab1Copies; i += blockDim.x) s_tab1[i] = gtab[i / kTab1Copies].x;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const unsigned tab1_addr = opaque_u32((unsigned)__cvta_generic_to_shared(s_tab1 + (lane & (kTab1Copies - 1))));
  const unsigned long long tid = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long wid = tid >> 5;
  unsigned long long its = 0;
  double acc = 0.0;
  for (int c = 0; c < cols; ++c) {
    const unsigned long long key = (wid * 100003ULL + c) * 64 + lane;
    const double s = 0.5 + 0.5 * u01(key * 3 + 1);
    const double guess = 24.0 + 160.0 * __shfl_sync(~0u, s, 0);
    double t[2], e[2], h[2], y[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      y[k] = 1.2 + 0.15 * u01(key * 7 + k);
      t[k] = guess;
      e[k] = exp(0.05 * guess);
      h[k] = e[k] + 0.01 * guess - y[k];
    }
    int left = 101;
    if (FAR) {
      float t0 = (float)t[0], t1 = (float)t[1], e0 = (float)e[0], e1 = (float)e[1];
      float h0 = (float)h[0], h1 = (float)h[1];
      const float y0 = (float)y[0], y1 = (float)y[1];
      while (fminf(fabsf(h0), fabsf(h1)) > kFar32H) {
        newton_far32_step(t0, e0, h0, y0);
        newton_far32_step(t1, e1, h1, y1);
        --left;
        ++its;
      }
      t[0] = t0;
      t[1] = t1;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        e[k] = exp_relaxed1(kRC, t[k], tab1_addr);
        h[k] = fma(0.01, t[k], e[k] - y[k]);
      }
    }
    do {
      if (abs_le_either(h[0], h[1], tol)) break;
      newton_relaxed_step(t[0], e[0], h[0], y[0], tab1_addr);
      newton_relaxed_step(t[1], e[1], h[1], y[1], tab1_addr);
      ++its;
    } while (--left);
    const int it = 101 - left;
    // finish the unconverged one (lockstep leftovers)
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      int itk = it;
      while (!abs_le(h[k], tol) && itk < 200) { newton_relaxed_step(t[k], e[k], h[k], y[k], tab1_addr); ++itk; }
      acc += t[k];
      if (counts) {
        const size_t idx = ((size_t)tid * cols + c) * 2 + k;
        counts[idx] = itk;
        roots[idx] = t[k];
      }
    }
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (lane == 0) atomicAdd(iters_out, its);
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::vector<double2> tab(kExpTableSize);
  for (int j = 0; j < kExpTableSize; ++j) {
    long double v = exp2l((long double)j / kExpTableSize);
    tab[j].x = (double)v;
    tab[j].y = (double)(v - (long double)tab[j].x);
  }
  double2* dtab;
  CK(cudaMalloc(&dtab, sizeof(double2) * kExpTableSize));
  CK(cudaMemcpy(dtab, tab.data(), sizeof(double2) * kExpTableSize, cudaMemcpyHostToDevice));
  unsigned long long* dits;
  CK(cudaMalloc(&dits, 8));
  double* sink;
  CK(cudaMalloc(&sink, sizeof(double) * 148 * 1024));
  const size_t smem = sizeof(double) * kExpTableSize * kTab1Copies;
  CK(cudaFuncSetAttribute(loop_k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(loop_k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int far = 0; far < 2; ++far) {
    for (int nw : {8, 12, 16, 20, 24, 32}) {
      const int cols = 64;
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaMemset(dits, 0, 8));
        cudaEventRecord(e0);
        if (far) loop_k<true><<<sms, nw * 32, smem>>>(dtab, cols, 1e-12, dits, sink, nullptr, nullptr);
        else loop_k<false><<<sms, nw * 32, smem>>>(dtab, cols, 1e-12, dits, sink, nullptr, nullptr);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long its = 0;
        CK(cudaMemcpy(&its, dits, 8, cudaMemcpyDeviceToHost));
        const double solves = (double)sms * nw * 32 * cols * 2;
        if (rep == 1)
          printf("far32 %d warps/SM %2d: %.3f ms, %.2f G solves/s, warp-iterations/solve-pair %.2f\n",
                 far, nw, ms, solves / (ms * 1e-3) / 1e9, (double)its / (sms * nw * cols));
      }
    }
  }
  // parity between the two variants on a big sample
  const int nw = 16, cols = 256;
  const size_t ns = (size_t)sms * nw * 32 * cols * 2;
  int *c0, *c1;
  double *r0, *r1;
  CK(cudaMalloc(&c0, ns * 4)); CK(cudaMalloc(&c1, ns * 4));
  CK(cudaMalloc(&r0, ns * 8)); CK(cudaMalloc(&r1, ns * 8));
  loop_k<false><<<sms, nw * 32, smem>>>(dtab, cols, 1e-12, dits, sink, c0, r0);
  loop_k<true><<<sms, nw * 32, smem>>>(dtab, cols, 1e-12, dits, sink, c1, r1);
  CK(cudaDeviceSynchronize());
  std::vector<int> h0(ns), h1(ns);
  std::vector<double> q0(ns), q1(ns);
  CK(cudaMemcpy(h0.data(), c0, ns * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h1.data(), c1, ns * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(q0.data(), r0, ns * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(q1.data(), r1, ns * 8, cudaMemcpyDeviceToHost));
  size_t flips = 0, bitdiff = 0;
  double maxrel = 0, mean = 0;
  for (size_t i = 0; i < ns; ++i) {
    flips += h0[i] != h1[i];
    bitdiff += q0[i] != q1[i];
    mean += h0[i];
    if (h0[i] == h1[i]) maxrel = fmax(maxrel, fabs(q0[i] - q1[i]) / fabs(q0[i]));
  }
  printf("parity: %zu solves, mean updates %.3f, count flips %zu, root bit diffs %zu, max rel root diff (same count) %.3g\n",
         ns, mean / ns, flips, bitdiff, maxrel);
  return 0;
}
