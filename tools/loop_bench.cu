// Design probe: throughput of the relaxed two-solve Newton loop alone (the
// deep worker's inner loop, colmath.cuh newton_relaxed_step) versus warps
// per SM, with realistic targets y ~ U(1.2, 1.35) and guesses 24 + 160 s,
// s ~ U(0.5, 1).  Prints ns per warp-iteration summed over the chip.
#include <cstdio>
#include <cstdlib>
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

template <int NS>
__global__ void loop_k(const double2* gtab, int cols, double tol, unsigned long long* iters_out, double* sink) {
  extern __shared__ double s_tab1[];
  for (int i = threadIdx.x; i < kExpTableSize * kTab1Copies; i += blockDim.x) s_tab1[i] = gtab[i / kTab1Copies].x;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const unsigned tab1_addr = opaque_u32((unsigned)__cvta_generic_to_shared(s_tab1 + (lane & (kTab1Copies - 1))));
  const unsigned long long wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  unsigned long long its = 0;
  double acc = 0.0;
  for (int c = 0; c < cols; ++c) {
    const unsigned long long key = (wid * 100003ULL + c) * 64 + lane;
    const double s = 0.5 + 0.5 * u01(key * 3 + 1);
    const double guess = 24.0 + 160.0 * __shfl_sync(~0u, s, 0);
    double t[NS], e[NS], h[NS], y[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      y[k] = 1.2 + 0.15 * u01(key * 7 + k);
      t[k] = guess;
      e[k] = exp(0.05 * guess);
      h[k] = e[k] + 0.01 * guess - y[k];
    }
    int left = 101;
    do {
      bool any = false;
#pragma unroll
      for (int k = 0; k < NS; ++k) any |= abs_le(h[k], tol);
      if (any) break;
#pragma unroll
      for (int k = 0; k < NS; ++k) newton_relaxed_step(t[k], e[k], h[k], y[k], tab1_addr);
      ++its;
    } while (--left);
#pragma unroll
    for (int k = 0; k < NS; ++k) acc += t[k];
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
  CK(cudaFuncSetAttribute(loop_k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(loop_k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int ns : {2, 4}) {
    for (int nw : {4, 8, 12, 16, 20, 24, 32}) {
      const int cols = 64;
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaMemset(dits, 0, 8));
        cudaEventRecord(e0);
        if (ns == 2) loop_k<2><<<sms, nw * 32, smem>>>(dtab, cols, 1e-12, dits, sink);
        else loop_k<4><<<sms, nw * 32, smem>>>(dtab, cols, 1e-12, dits, sink);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long its = 0;
        CK(cudaMemcpy(&its, dits, 8, cudaMemcpyDeviceToHost));
        if (rep == 1)
          printf("solves/lane %d warps/SM %2d: %.3f ms, warp-iterations %llu, %.3f ns/warp-iter (chip), %.1f Gupd/s\n",
                 ns, nw, ms, its, ms * 1e6 / its, (double)its * 32 * ns / (ms * 1e-3) / 1e9);
      }
    }
  }
  return 0;
}
