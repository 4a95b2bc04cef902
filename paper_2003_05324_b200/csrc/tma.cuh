// mbarrier / TMA (cp.async.bulk.tensor) helpers shared by the tcgen05 and
// DMMA update kernels, plus host-side tensor-map encoding.
#pragma once
#include <cuda.h>
#include <stdint.h>

#include "mt_grid.cuh"

namespace mt_tma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// relaxed arrive: no release fence, so it does not wait for this thread's
// outstanding global stores (a default .release arrive compiles to
// MEMBAR.ALL.CTA, which stalls an epilogue warp on its own C stores).  Use only
// where the barrier orders on-chip state (TMEM reads finished via
// tcgen05.wait::ld, or smem reads whose values the caller already consumed).
__device__ __forceinline__ void mbar_arrive_relaxed(uint64_t* b) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)map) : "memory");
}

// host: 2D row-major matrix of `rows` x `cols` elements (elem bytes `es`),
// box `box_cols` x `box_rows`, with the given swizzle
int make_map_2d(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int es,
                int box_cols, int box_rows, CUtensorMapSwizzle swz);

}  // namespace mt_tma
