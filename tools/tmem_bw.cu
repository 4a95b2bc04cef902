// TMEM -> register read throughput on one SM (dev microbenchmark):
// W warps (2..16), each reading its lane quadrant with tcgen05.ld 32x32b.x32,
// NL loads in flight per tcgen05.wait::ld.  Prints bytes per SM clock.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_bw tools/tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define LD32(v, addr)                                                                              \
  asm volatile(                                                                                    \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"     \
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"          \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),        \
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),    \
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), \
        "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), \
        "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])                                         \
      : "r"(addr))

template <int NL>
__global__ void tmem_read(int iters, unsigned long long* cyc, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
  const int colw = (warp >> 2) * 128;  // warps beyond 4 read other columns
  float acc = 0.f;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t v[NL][32];
#pragma unroll
    for (int l = 0; l < NL; ++l) LD32(v[l], base + ((colw + l * 32 + it * 32) & 511));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int l = 0; l < NL; ++l)
#pragma unroll
      for (int u = 0; u < 32; ++u) acc += __uint_as_float(v[l][u]);
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int NL>
void run(int warps) {
  const int iters = 4096, ctas = 148;
  unsigned long long* cyc;
  float* sink;
  cudaMalloc(&cyc, ctas * 8);
  cudaMalloc(&sink, ctas * warps * 32 * 4);
  tmem_read<NL><<<ctas, warps * 32>>>(iters, cyc, sink);
  tmem_read<NL><<<ctas, warps * 32>>>(iters, cyc, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double bytes = (double)iters * warps * NL * 32 * 32 * 4;
  printf("warps %2d loads/wait %d: %.1f B/clk/SM (%s)\n", warps, NL, bytes / (double)h[0],
         cudaGetErrorString(e));
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<1>(w);
    run<2>(w);
    run<4>(w);
  }
  return 0;
}
