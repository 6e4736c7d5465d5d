// Dependent-chain latencies of the FP64 ops the Newton loop uses (1 warp).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_lat(double* out, long long* cyc, int n, double a, double b) {
  double x = threadIdx.x * 1e-9 + 1.0, y = 1.0;
  __shared__ double2 tab[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) tab[i] = make_double2(1.0 + i * 1e-9, 0);
  __syncthreads();
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  t1 = clock64(); cyc[0] = t1 - t0;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, b);
  t1 = clock64(); cyc[1] = t1 - t0;
  // MUFU.RCP64H chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) { asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(y)); }
  t1 = clock64(); cyc[2] = t1 - t0;
  // LDS chain (index from data)
  int idx = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { double2 v = tab[idx & 511]; idx = (int)(v.x) + (idx >> 1); }
  t1 = clock64(); cyc[3] = t1 - t0;
  // DSETP + branch-ish chain: compare result feeding select
  t0 = clock64();
  for (int i = 0; i < n; ++i) { x = (fabs(x) <= a) ? x + b : x - b; }
  t1 = clock64(); cyc[4] = t1 - t0;
  out[threadIdx.x] = x + y + idx;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64);
  const int n = 4096;
  k_lat<<<1, 32>>>(o, c, n, 0.999999, 1e-9);
  k_lat<<<1, 32>>>(o, c, n, 0.999999, 1e-9);
  long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
  const char* nm[5] = {"dfma", "dadd", "mufu_rcp64h", "lds128_dep", "dsetp_sel_dadd"};
  for (int i = 0; i < 5; ++i) printf("{\"op\": \"%s\", \"cycles_per_op\": %.2f}\n", nm[i], (double)h[i] / n);
  return 0;
}
