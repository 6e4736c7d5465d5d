// zc_probe.cu -- feasibility probe for the sparse D2H of the host-buffer path:
// (1) host zero-fill bandwidth over pinned memory with T threads, (2) a copy
// kernel writing device rows straight into mapped pinned host memory at a
// given segment size and density, (3) both together with a concurrent H2D DMA
// of the step's inputs.  nvcc -O2 -arch=sm_100a -o tools/zc_probe tools/zc_probe.cu -lpthread
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

// segment s (seg_bytes each) is copied when keep[s] != 0; one warp per 32 x 16 B
__global__ void sparse_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, const unsigned char* __restrict__ keep,
                            size_t n16, int seg16) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    if (keep[i / seg16]) dst[i] = src[i];
  }
}

static void zero_mt(char* p, size_t bytes, int T, const unsigned char* keep, size_t seg) {
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t)
    th.emplace_back([=] {
      size_t nseg = bytes / seg, a = nseg * t / T, b = nseg * (t + 1) / T;
      if (!keep) { memset(p + a * seg, 0, (b - a) * seg); return; }
      // runs of not-kept segments
      size_t s = a;
      while (s < b) {
        while (s < b && keep[s]) ++s;
        size_t e = s;
        while (e < b && !keep[e]) ++e;
        if (e > s) memset(p + s * seg, 0, (e - s) * seg);
        s = e;
      }
    });
  for (auto& x : th) x.join();
}

int main(int argc, char** argv) {
  const size_t out_bytes = 879ull << 20, in_bytes = 432ull << 20;
  char *h_out, *h_in, *d_out, *d_in;
  CK(cudaHostAlloc(&h_out, out_bytes, cudaHostAllocDefault));
  CK(cudaHostAlloc(&h_in, in_bytes, cudaHostAllocDefault));
  CK(cudaMalloc(&d_out, out_bytes));
  CK(cudaMalloc(&d_in, in_bytes));
  memset(h_out, 1, out_bytes);
  memset(h_in, 1, in_bytes);
  CK(cudaMemset(d_out, 2, out_bytes));
  int ncpu = std::thread::hardware_concurrency();
  printf("cpus %d\n", ncpu);
  for (int T : {1, 4, 8, 12, 16, 32}) {
    if (T > ncpu) break;
    double best = 1e9;
    for (int r = 0; r < 3; ++r) { double t = now(); zero_mt(h_out, out_bytes, T, nullptr, 4096); best = std::min(best, now() - t); }
    printf("memset %2d threads: %.1f GB/s (%.2f ms / 879 MiB)\n", T, out_bytes / best / 1e9, best * 1e3);
  }
  cudaStream_t s1, s2;
  CK(cudaStreamCreate(&s1));
  CK(cudaStreamCreate(&s2));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timed = [&](auto fn) { float best = 1e9; for (int r = 0; r < 4; ++r) { CK(cudaEventRecord(e0, s1)); fn(); CK(cudaEventRecord(e1, s1)); CK(cudaEventSynchronize(e1)); float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); best = std::min(best, ms); } return best; };
  float ms = timed([&] { CK(cudaMemcpyAsync(h_out, d_out, out_bytes, cudaMemcpyDeviceToHost, s1)); });
  printf("DMA d2h dense: %.2f ms (%.1f GB/s)\n", ms, out_bytes / ms / 1e6);
  ms = timed([&] { CK(cudaMemcpyAsync(d_in, h_in, in_bytes, cudaMemcpyHostToDevice, s1)); });
  printf("DMA h2d dense: %.2f ms (%.1f GB/s)\n", ms, in_bytes / ms / 1e6);
  unsigned char* keep_h;
  unsigned char* keep_d;
  for (int seg : {32, 64, 128, 256, 512, 2048}) {
    for (double dens : {1.0, 0.57, 0.3}) {
      size_t nseg = out_bytes / seg;
      CK(cudaHostAlloc(&keep_h, nseg, cudaHostAllocDefault));
      CK(cudaMalloc(&keep_d, nseg));
      // clustered keeps: runs of ~8 segments
      unsigned long long x = 88172645463325252ull;
      size_t kept = 0;
      for (size_t s = 0; s < nseg;) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        bool k = (x % 1000) < dens * 1000;
        size_t run = 1 + (x >> 20) % 15;
        for (size_t j = 0; j < run && s < nseg; ++j, ++s) { keep_h[s] = k; kept += k; }
      }
      CK(cudaMemcpy(keep_d, keep_h, nseg, cudaMemcpyHostToDevice));
      for (int blocks : {148 * 2, 148 * 8}) {
        ms = timed([&] { sparse_copy<<<blocks, 256, 0, s1>>>((const uint4*)d_out, (uint4*)h_out, keep_d, out_bytes / 16, seg / 16); });
        printf("zero-copy seg %4d B density %.2f blocks %4d: %.2f ms, %.1f GB/s of kept bytes (%.0f MB)\n", seg, dens, blocks, ms,
               kept * (double)seg / ms / 1e6, kept * (double)seg / 1e6);
      }
      if (seg == 128 && dens < 1.0) {
        // combined: H2D DMA + zero-copy sparse + host zero-fill of the rest
        for (int T : {4, 8, 12, 15}) {
          if (T > ncpu) break;
          double best = 1e9;
          for (int r = 0; r < 3; ++r) {
            CK(cudaDeviceSynchronize());
            double t = now();
            CK(cudaMemcpyAsync(d_in, h_in, in_bytes, cudaMemcpyHostToDevice, s2));
            sparse_copy<<<148 * 8, 256, 0, s1>>>((const uint4*)d_out, (uint4*)h_out, keep_d, out_bytes / 16, seg / 16);
            double t1 = now();
            zero_mt(h_out, out_bytes, T, keep_h, seg);
            double t2 = now();
            CK(cudaDeviceSynchronize());
            double t3 = now();
            if (t3 - t < best) { best = t3 - t; printf("  combined T=%d: launch %.2f, zero-fill %.2f ms, total %.2f ms\n", T, (t1 - t) * 1e3, (t2 - t1) * 1e3, (t3 - t) * 1e3); }
          }
        }
      }
      CK(cudaFreeHost(keep_h));
      CK(cudaFree(keep_d));
    }
  }
  return 0;
}
