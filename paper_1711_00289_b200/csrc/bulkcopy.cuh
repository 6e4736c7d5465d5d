// bulkcopy.cuh -- small PTX helpers: shared-memory addresses, the
// warp-per-column kernel's cp.async group-entry prefetch, the 256-bit global
// store of a 4-column group row, and the 16-byte cp.async of the tiled shallow
// kernel.
#pragma once
#include <cstdint>

namespace cvg {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

// A shared-memory address the compiler cannot rematerialise (it would
// otherwise recompute it from %cgactaid inside loops under register caps).
__device__ __forceinline__ unsigned opaque_u32(unsigned x) {
  asm volatile("mov.b32 %0, %0;" : "+r"(x));
  return x;
}
// 8-byte cp.async global -> shared (dst as a shared-window address).
__device__ __forceinline__ void cp_async8_u32(unsigned dst_smem, const void* src_gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst_smem), "l"(src_gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// 256-bit global store (sm_100: STG.E.ENL2.256); p 32-byte aligned.
__device__ __forceinline__ void st_global_v4f64(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

// 16-byte cp.async global -> shared, L1 bypassed (both 16-byte aligned).
__device__ __forceinline__ void cp_async16_u32(unsigned dst_smem, const void* src_gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst_smem), "l"(src_gmem) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace cvg
