// FP64 pipe microbenchmark for the roofline denominator (B200, sm_100a).
// Each thread runs NCHAIN independent dependent chains so the FP64 pipe,
// not latency, bounds issue.  Prints one JSON line per probe.
#include <cstdio>
#include <cuda_runtime.h>

#define NCHAIN 8
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[NCHAIN];
  for (int c = 0; c < NCHAIN; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < NCHAIN; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0; for (int c = 0; c < NCHAIN; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dadd(double* out, int iters, double a, double b) {
  double x[NCHAIN];
  for (int c = 0; c < NCHAIN; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < NCHAIN; ++c) x[c] = __dadd_rn(x[c], a);
  }
  double s = 0; for (int c = 0; c < NCHAIN; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dmul(double* out, int iters, double a, double b) {
  double x[NCHAIN];
  for (int c = 0; c < NCHAIN; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < NCHAIN; ++c) x[c] = __dmul_rn(x[c], a);
  }
  double s = 0; for (int c = 0; c < NCHAIN; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ddiv(double* out, int iters, double a, double b) {
  double x[NCHAIN];
  for (int c = 0; c < NCHAIN; ++c) x[c] = threadIdx.x * 1e-3 + c + 1.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < NCHAIN; ++c) x[c] = a / x[c] + b;
  }
  double s = 0; for (int c = 0; c < NCHAIN; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_exp(double* out, int iters, double a, double b) {
  double x[NCHAIN];
  for (int c = 0; c < NCHAIN; ++c) x[c] = threadIdx.x * 1e-3 + c * 0.1;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < NCHAIN; ++c) x[c] = exp(x[c]) * a;
  }
  double s = 0; for (int c = 0; c < NCHAIN; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_sin(double* out, int iters, double a, double b) {
  double x[NCHAIN];
  for (int c = 0; c < NCHAIN; ++c) x[c] = threadIdx.x * 1e-3 + c * 0.1;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < NCHAIN; ++c) x[c] = sin(x[c]) * a + b;
  }
  double s = 0; for (int c = 0; c < NCHAIN; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

typedef void (*kfn)(double*, int, double, double);

static int run(const char* name, kfn f, int blocks, int threads, int iters,
               double a, double b, double ops_per_iter_lane, double* out) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  for (int w = 0; w < 3; ++w) f<<<blocks, threads>>>(out, iters, a, b);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    CK(cudaEventRecord(e0));
    f<<<blocks, threads>>>(out, iters, a, b);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  double lanes = (double)blocks * threads;
  double ops = lanes * iters * NCHAIN * ops_per_iter_lane;
  printf("{\"probe\": \"%s\", \"ms\": %.4f, \"Gop_per_s\": %.1f, \"blocks\": %d, \"threads\": %d}\n",
         name, best, ops / (best * 1e-3) / 1e9, blocks, threads);
  return 0;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz\": %d}\n", p.name, p.multiProcessorCount, clk);
  int sms = p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, (size_t)sms * 64 * 1024 * sizeof(double)));
  // flops: a DFMA is 2 flops; report "Gop" = FP64 lane-instructions/s and DFMA GFLOP/s = 2x.
  for (int tpb : {256, 512}) {
    int blocks = sms * (2048 / tpb);
    run("dfma_inst", k_dfma, blocks, tpb, 4096, 0.999999, 1e-7, 1.0, out);
    run("dadd_inst", k_dadd, blocks, tpb, 4096, 1e-7, 0, 1.0, out);
    run("dmul_inst", k_dmul, blocks, tpb, 4096, 0.9999999, 0, 1.0, out);
  }
  int blocks = sms * 8;
  run("ddiv_per_s", k_ddiv, blocks, 256, 512, 1.5, 1.0, 1.0, out);
  run("exp_per_s", k_exp, blocks, 256, 512, 0.5, 0, 1.0, out);
  run("sin_per_s", k_sin, blocks, 256, 512, 0.9, 0.1, 1.0, out);
  return 0;
}
