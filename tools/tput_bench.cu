// Throughput of MUFU.RCP64H, DSETP and the mixed Newton-loop op mix (all SMs).
#include <cstdio>
#include <cuda_runtime.h>
#define NC 8
__global__ void k_rcp(double* out, int n) {
  double x[NC];
  for (int c = 0; c < NC; ++c) x[c] = 1.0 + threadIdx.x * 1e-6 + c;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < NC; ++c) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(x[c]));
  double s = 0; for (int c = 0; c < NC; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dsetp(double* out, int n, double t) {
  double x[NC]; int cnt = 0;
  for (int c = 0; c < NC; ++c) x[c] = 1.0 + threadIdx.x * 1e-6 + c;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < NC; ++c) { int p; asm volatile("{.reg .pred q; setp.le.f64 q, %1, %2; selp.s32 %0, 1, 0, q;}" : "=r"(p) : "d"(x[c]), "d"(t)); cnt += p; x[c] += 1e-300; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = cnt + x[0];
}
__global__ void k_lds(double* out, int n) {
  __shared__ double2 tab[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) tab[i] = make_double2(i, 0);
  __syncthreads();
  int idx[NC]; double s = 0;
  for (int c = 0; c < NC; ++c) idx[c] = threadIdx.x * 7 + c * 13;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < NC; ++c) { double2 v = tab[idx[c] & 511]; s += v.y; idx[c] += (int)v.x & 3; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + idx[0];
}
typedef void (*kf)(double*, int);
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o; cudaMalloc(&o, sms * 2048 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256, n = 1024;
  auto time = [&](const char* name, auto launch, double ops_per_thread) {
    launch(); launch(); cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    double lanes = (double)blocks * threads * ops_per_thread;
    printf("{\"op\": \"%s\", \"Glane_ops_per_s\": %.1f, \"warp_cycles_per_instr_per_smsp\": %.2f}\n", name, lanes / (best * 1e-3) / 1e9, (sms * 4 * 1.965e9 * best * 1e-3) / (lanes / 32));
  };
  time("mufu_rcp64h", [&] { k_rcp<<<blocks, threads>>>(o, n); }, (double)n * NC);
  time("dsetp(+dadd)", [&] { k_dsetp<<<blocks, threads>>>(o, n, 0.5); }, (double)n * NC);
  time("lds128(+dadd+iadd)", [&] { k_lds<<<blocks, threads>>>(o, n); }, (double)n * NC);
  return 0;
}
