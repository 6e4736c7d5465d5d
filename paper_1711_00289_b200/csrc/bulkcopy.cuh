// bulkcopy.cuh -- small PTX helpers: shared-memory addresses, the
// warp-per-column kernel's cp.async group-entry prefetch, the 256-bit global
// store of a 4-column group row, and the tile loads of the tiled shallow
// kernel (TMA tensor tiles; 16-byte cp.async as the fallback).
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

// mbarrier (8 bytes of shared memory) + TMA tensor-tile load: the tiled
// shallow kernel fetches a [L][32] box of a level-major field with ONE
// instruction (cp.async.bulk.tensor.2d), completion counted on the barrier.
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@p bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(bar), "r"(parity) : "memory");
}
// box (x0.., y0..) of the 2-D tensor described by tmap -> shared memory
__device__ __forceinline__ void tma_load_2d(unsigned dst_smem, const void* tmap, int x0, int y0, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst_smem),
      "l"(tmap), "r"(x0), "r"(y0), "r"(bar)
      : "memory");
}

}  // namespace cvg
