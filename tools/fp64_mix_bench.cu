// FP64 pipe throughput vs operand form: DFMA with register operands
// (3 distinct vector registers) vs uniform/immediate operands, and the
// Newton fast-path loop itself (no memory, warp-uniform data).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1711_00289_b200/csrc/colmath.cuh"
#define NC 8
using namespace cvg;
__global__ void k_reg3(double* out, int n) {
  double x[NC], y[NC], z[NC];
  for (int c = 0; c < NC; ++c) { x[c] = threadIdx.x * 1e-9 + c; y[c] = 0.999999 + c * 1e-9; z[c] = 1e-9 * c; }
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < NC; ++c) x[c] = fma(x[c], y[c], z[c]);
#pragma unroll
    for (int c = 0; c < NC; ++c) z[c] = fma(z[c], y[c], x[c]);
  }
  double s = 0; for (int c = 0; c < NC; ++c) s += x[c] + z[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_newton(double* out, int n, int nsolve, const double2* gtab) {
  extern __shared__ double2 tab[];
  for (int i = threadIdx.x; i < 512 * 8; i += blockDim.x) tab[i] = gtab[i / 8];
  __syncthreads();
  const double2* mt = tab + (threadIdx.x & 7);
  double acc = 0;
  for (int r = 0; r < nsolve; ++r) {
    double t[4], e[4], h[4], y[4];
    for (int s = 0; s < 4; ++s) {
      y[s] = 1.25 + 1e-3 * ((threadIdx.x + s * 7) & 31);
      t[s] = 150.0 + r * 1e-3;
      e[s] = exp005_tang<8>(t[s], mt);
      h[s] = sub(add(e[s], mul(kMC.c001, t[s])), y[s]);
    }
    for (int it = 0; it < n; ++it) {
#pragma unroll
      for (int s = 0; s < 4; ++s) t[s] = sub(t[s], div_fast(h[s], add(mul(kMC.c005, e[s]), kMC.c001)));
#pragma unroll
      for (int s = 0; s < 4; ++s) e[s] = exp005_tang<8>(t[s], mt);
#pragma unroll
      for (int s = 0; s < 4; ++s) h[s] = sub(add(e[s], mul(kMC.c001, t[s])), y[s]);
    }
    acc += t[0] + t[1] + t[2] + t[3];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o; cudaMalloc(&o, sms * 2048 * 8);
  double2 htab[512]; for (int j = 0; j < 512; ++j) { long double v = exp2l((long double)j / 512); htab[j] = make_double2((double)v, (double)(v - (long double)(double)v)); }
  double2* dtab; cudaMalloc(&dtab, sizeof(htab)); cudaMemcpy(dtab, htab, sizeof(htab), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaFuncSetAttribute(k_newton, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  auto timeit = [&](auto launch) { launch(); cudaDeviceSynchronize(); float best = 1e9; for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; } return best; };
  for (int tpb : {256, 512, 1024}) {
    int blocks = sms * (2048 / tpb);
    float ms = timeit([&] { k_reg3<<<blocks, tpb>>>(o, 1024); });
    double lanes = (double)blocks * tpb * 1024 * NC * 2;
    printf("{\"probe\": \"dfma_3reg\", \"tpb\": %d, \"G_dfma_per_s\": %.1f}\n", tpb, lanes / (ms * 1e-3) / 1e9);
  }
  for (int warps : {4, 8, 12, 16, 24, 32}) {
    int tpb = warps * 32;
    float ms = timeit([&] { k_newton<<<sms, tpb, 65536>>>(o, 12, 16, dtab); });
    double upd = (double)sms * tpb * 16 * 12 * 4;
    // FP64 instrs per update in the fast loop: 25 (2 deriv + 8 div + 1 t + 11 exp incl x + 3 h)
    printf("{\"probe\": \"newton4_fastloop\", \"warps_per_sm\": %d, \"G_upd_per_s\": %.1f, \"fp64_pipe_frac_est\": %.3f}\n",
           warps, upd / (ms * 1e-3) / 1e9, upd * 25 / (ms * 1e-3) / 18.4e12);
  }
  return 0;
}
