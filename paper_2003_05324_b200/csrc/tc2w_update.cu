// Bulk off-band FP32 trailing update on CTA pairs with FULL-WIDTH work items:
// each pair computes a 256 x 512 block (two M=256, N=256 tcgen05.mma.cta_group::2
// per product, 3xTF32) so every staged A row feeds twice the MMA work.
//
//   C_ij <- C_ij - A_ik A_jk^T      (kernels.gemm FP32 path, factor.py:273-274)
//
// Why: in the 256 x 256-item pair kernel (tc2_update.cu) the MMA issuer, not
// the epilogue, waits -- on TMA operand delivery (~42 B/clk/SM at full MMA
// rate, the L2->SM limit).  A 256 x 512 item stages 48 KB per 16-wide K slab
// for 1536 MMA cycles (32 B/clk/SM).  The price: the two N=256 accumulators
// fill TMEM (512 columns), so TMEM is single-buffered and the MMA waits for
// the (TMA-streamed, short) epilogue of the previous item; the producer keeps
// prefetching the next item's slabs meanwhile.
//
// Same arithmetic per output element as tc2_update.cu / tc_update.cu (K slabs
// in order; per 8-wide K step lo*hi, hi*lo, hi*hi into one accumulator), so
// results are bit-identical to them (tests/test_gpu_tc.py).  Used for the bulk
// update when nb % 512 == 0 (option 12); panel-column updates and TRSMs stay
// on tc2_update.cu.
#include <cuda.h>

#include "tma.cuh"
#include "tc2_common.cuh"

namespace {
using namespace mt_tma;
using namespace mt_pair;

constexpr int BM = 128;     // accumulator rows per CTA (pair M = 256)
constexpr int BNM = 256;    // N of one MMA
constexpr int BNI = 512;    // N of a work item (two MMAs per product)
constexpr int BNH = 128;    // rows of B each CTA stages per MMA half
#ifndef MT_TC2W_STAGES
#define MT_TC2W_STAGES 3
#endif
#ifndef MT_TC2W_EPIW
#define MT_TC2W_EPIW 4
#endif
constexpr int BK = 16, STAGES = MT_TC2W_STAGES;
constexpr int A_BYTES = BM * BK * 4;    // 8 KB
constexpr int BH_BYTES = BNH * BK * 4;  // 8 KB per half
constexpr int HALF = A_BYTES + 2 * BH_BYTES;  // hi or lo part of a stage: 24 KB
constexpr int STAGE_BYTES = 2 * HALF;         // 48 KB
// epilogue warps: 4 (one per TMEM lane quadrant) or 8 (two per quadrant, each
// draining half of the item's columns)
constexpr int EPI_WARPS = MT_TC2W_EPIW;
constexpr int NUM_THREADS = 64 + 32 * EPI_WARPS;
#ifndef MT_TC2W_CSLOTS
#define MT_TC2W_CSLOTS 4
#endif
constexpr int CSLOTS = MT_TC2W_CSLOTS, CSLOT_BYTES = 32 * 32 * 4;  // loads CSLOTS-1 chunks ahead
constexpr int EPI_BYTES = EPI_WARPS * CSLOTS * CSLOT_BYTES;  // 64 KB at 4 slots
constexpr int TMEM_COLS = 512;  // one 128 x 512 accumulator per CTA
constexpr int SCHED = 4;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 640;
static_assert(SMEM_BYTES <= 232448, "shared memory");

// kind::tf32, D f32, A/B tf32 K-major, N = 256, M = 256 (cta_group::2)
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BNM >> 3) << 17) |
                            ((uint32_t)(256 >> 4) << 24);

__device__ __forceinline__ void umma2(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}

struct WorkW {
  int64_t slot0;
  int nitems;    // slots * nsubm (256 x 512 items)
  int nsubm;
  int* counter;  // [work queue head, unused]
  unsigned long long* span;
  int l2pf;      // stage each warp's C rows in L2 at item start (option 13)
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    tc2w_update_kernel(Grid g, int k, WorkW w, const __grid_constant__ CUtensorMap map_a,
                       const __grid_constant__ CUtensorMap map_b,
                       const __grid_constant__ CUtensorMap map_c) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* epi = smem + STAGES * STAGE_BYTES;
  uint64_t* full = (uint64_t*)(epi + EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // single accumulator buffer
  uint64_t* tempty = tfull + 1;
  uint64_t* sfull = tempty + 1;
  uint64_t* sempty = sfull + SCHED;
  int* sitem = (int*)(sempty + SCHED);
  int* si = sitem + SCHED;
  int* sj = si + SCHED;
  uint64_t* cbar = (uint64_t*)(sj + SCHED);
  uint32_t* tmem_slot = (uint32_t*)(cbar + EPI_WARPS * CSLOTS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // co-scheduled band update
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const int nb = g.nb;
  const int ksteps = nb / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 2 * EPI_WARPS);
    for (int s = 0; s < SCHED; ++s) {
      mbar_init(&sfull[s], 1);
      mbar_init(&sempty[s], 2 + 2 * EPI_WARPS);
    }
    for (int s = 0; s < EPI_WARPS * CSLOTS; ++s) mbar_init(&cbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (w.span && threadIdx.x == 0) atomicMin(&w.span[0], mt_globaltimer());
  const uint32_t tmem_base = *tmem_slot;

  auto next_item = [&](uint32_t li, int* pi, int* pj) {
    const int s = li % SCHED;
    mbar_wait_cl(&sfull[s], (li / SCHED) & 1);
    const int item = *(volatile int*)&sitem[s];
    int dep = item;
    if (pi) {
      *pi = *(volatile int*)&si[s];
      *pj = *(volatile int*)&sj[s];
      dep ^= *pi ^ *pj;
    }
    dep = __reduce_xor_sync(0xffffffffu, dep);
    if ((threadIdx.x & 31) == 0 && dep != 0x7fffffff) {
      if (leader) mbar_arrive_relaxed(&sempty[s]);
      else mbar_arrive_cl_relaxed(peer_addr(&sempty[s], 0));
    }
    return item;
  };

  if (warp == 0) {
    // ------------------------------------------------ work queue + TMA producer
    if (lane == 0) {
      uint32_t it = 0;
      for (uint32_t li = 0;; ++li) {
        const int s = li % SCHED;
        int item, i = 0, j = 0;
        if (leader) {
          mbar_wait(&sempty[s], ((li / SCHED) & 1) ^ 1);
          if (g.failed()) {
            item = -1;
          } else {
            item = atomicAdd(w.counter, 1);
            if (item >= w.nitems) item = -1;
          }
          if (item >= 0) g.off_slot_ij(w.slot0 + item / w.nsubm, i, j);
          sitem[s] = item; si[s] = i; sj[s] = j;
          st_cl_u32(peer_addr(&sitem[s], 1), (uint32_t)item);
          st_cl_u32(peer_addr(&si[s], 1), (uint32_t)i);
          st_cl_u32(peer_addr(&sj[s], 1), (uint32_t)j);
          mbar_arrive(&sfull[s]);
          mbar_arrive_cl(peer_addr(&sfull[s], 1));
        } else {
          mbar_wait_cl(&sfull[s], (li / SCHED) & 1);
          item = *(volatile int*)&sitem[s];
          i = *(volatile int*)&si[s];
          j = *(volatile int*)&sj[s];
          if ((item ^ i ^ j) != 0x7fffffff) mbar_arrive_cl_relaxed(peer_addr(&sempty[s], 0));
        }
        if (item < 0) break;
        const int m0 = (item % w.nsubm) * (2 * BM) + (int)rank * BM;
        const int arow = (int)g.split_row(i, k) + m0;
        const int brow = (int)g.split_row(j, k) + (int)rank * BNH;  // + h * 256
        for (int ks = 0; ks < ksteps; ++ks, ++it) {
          const int st = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty[st], ph ^ 1);
          unsigned char* sb = smem + st * STAGE_BYTES;
          if (leader) mbar_expect_tx(&full[st], 2 * STAGE_BYTES);
          const uint32_t bar = peer_addr(&full[st], 0);
          // [A hi | B hi h0 | B hi h1 | A lo | B lo h0 | B lo h1]
          tma_load_pair(sb, &map_a, bar, ks * BK, arow);
          tma_load_pair(sb + A_BYTES, &map_b, bar, ks * BK, brow);
          tma_load_pair(sb + A_BYTES + BH_BYTES, &map_b, bar, ks * BK, brow + BNM);
          tma_load_pair(sb + HALF, &map_a, bar, ks * BK, arow + nb);
          tma_load_pair(sb + HALF + A_BYTES, &map_b, bar, ks * BK, brow + nb);
          tma_load_pair(sb + HALF + A_BYTES + BH_BYTES, &map_b, bar, ks * BK, brow + BNM + nb);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (leader only)
    if (leader) {
      uint32_t it = 0;
      for (uint32_t li = 0;; ++li) {
        const int item = next_item(li, nullptr, nullptr);
        if (item < 0) break;
        mbar_wait_cl(tempty, (li & 1) ^ 1);  // previous item's accumulator drained
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int ks = 0; ks < ksteps; ++ks, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (lane == 0) {
            unsigned char* st = smem + s * STAGE_BYTES;
            const unsigned char* ahi = st;
            const unsigned char* alo = st + HALF;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const unsigned char* bhi = st + A_BYTES + h * BH_BYTES;
              const unsigned char* blo = st + HALF + A_BYTES + h * BH_BYTES;
              const uint32_t dcol = tmem_base + h * BNM;
#pragma unroll
              for (int kk = 0; kk < BK / 8; ++kk) {
                const int off = kk * 32;
                const uint32_t first = (ks == 0 && kk == 0) ? 0u : 1u;
                umma2(dcol, sw64_desc(alo + off), sw64_desc(bhi + off), first);
                umma2(dcol, sw64_desc(ahi + off), sw64_desc(blo + off), 1u);
                umma2(dcol, sw64_desc(ahi + off), sw64_desc(bhi + off), 1u);
              }
            }
            umma2_commit_both(&empty[s]);
            if (ks == ksteps - 1) umma2_commit_both(tfull);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ------------------------------------------------ TMA epilogue (warps 2..5, both CTAs)
    const int q = warp & 3;
    unsigned char* wslots = epi + (warp - 2) * CSLOTS * CSLOT_BYTES;
    uint64_t* wbar = cbar + (warp - 2) * CSLOTS;
    uint32_t gl = 0, gu = 0;
    const uint32_t tempty_leader = peer_addr(tempty, 0);
    constexpr int NCH = BNI / 32 / (EPI_WARPS / 4);  // chunks of 32 columns per warp and item
    const int cbase = ((warp - 2) / 4) * NCH;        // this warp's first chunk
    for (uint32_t li = 0;; ++li) {
      int i, j;
      const int item = next_item(li, &i, &j);
      if (item < 0) break;
      const int m0 = (item % w.nsubm) * (2 * BM) + (int)rank * BM;
      const int crow = (int)((g.scol(j) + (i - j - g.t)) * (int64_t)nb) + m0 + q * 32;
      auto load_chunk = [&](int c, int newer) {
        if (lane == 0) {
          if (newer >= 4) bulk_wait_read<4>();
          else if (newer == 3) bulk_wait_read<3>();
          else if (newer == 2) bulk_wait_read<2>();
          else if (newer == 1) bulk_wait_read<1>();
          else bulk_wait_read<0>();
          const uint32_t s = gl % CSLOTS;
          mbar_expect_tx(&wbar[s], CSLOT_BYTES);
          tma_load_2d(wslots + s * CSLOT_BYTES, &map_c, &wbar[s], (cbase + c) * 32, crow);
        }
        ++gl;
      };
      for (int c = 0; c < CSLOTS - 1; ++c) load_chunk(c, (int)gu - (int)gl + CSLOTS - 1);
      if (w.l2pf && lane == 0 && cbase == 0) {
        // the TMEM drain is on the MMA's critical path (single-buffered): stage the
        // rest of this warp's C rows (32 x 2 KB) in L2 while the MMAs run
        const float* crow_p = g.stile(i, j) + (int64_t)(m0 + q * 32) * nb;
        for (int r = 0; r < 32; ++r)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(crow_p + (int64_t)r * nb),
                       "r"(nb * 4)
                       : "memory");
      }
      mbar_wait(tfull, li & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < NCH; ++c) {
        uint32_t v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
            "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
              "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
              "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
              "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
              "=r"(v[31])
            : "r"(taddr + (cbase + c) * 32));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c == NCH - 1) {
          // the whole accumulator is in registers now: let the next item's MMAs start
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) mbar_arrive_cl_relaxed(tempty_leader);
        }
        const uint32_t s = gu % CSLOTS;
        mbar_wait(&wbar[s], (gu / CSLOTS) & 1);
        const uint32_t row = smem_u32(wslots + s * CSLOT_BYTES) + lane * 128;
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          const uint32_t a = row + ((x ^ (lane & 7)) << 4);
          float4 cc = lds128(a);
          cc.x -= __uint_as_float(v[4 * x]);
          cc.y -= __uint_as_float(v[4 * x + 1]);
          cc.z -= __uint_as_float(v[4 * x + 2]);
          cc.w -= __uint_as_float(v[4 * x + 3]);
          sts128(a, cc);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&map_c, wslots + s * CSLOT_BYTES, (cbase + c) * 32, crow);
          bulk_commit();
        }
        ++gu;
        if (c + CSLOTS - 1 < NCH) load_chunk(c + CSLOTS - 1, (int)gu - (int)gl + CSLOTS - 1);
      }
    }
    if (lane == 0) bulk_wait_all();
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  if (w.span && threadIdx.x == 0) atomicMax(&w.span[1], mt_globaltimer());
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

int g_smw = 0;

}  // namespace

bool mt_tc2w_supported(const Grid& g) { return g.nb % BNI == 0; }

// bulk update of step k over off-band slots [s0, s0 + scnt); `ctas` caps the grid
int mt_tc2w_launch(const Grid& g, int k, int64_t s0, int64_t scnt, int ctas, cudaStream_t st,
                   unsigned long long* span) {
  if (scnt <= 0) return MT_OK;
  CUtensorMap ma, mb, mc;
  const int64_t split_rows = g.split_rows();
  int rc = make_map_2d(&ma, g.split, split_rows, g.nb, 4, BK, BM, CU_TENSOR_MAP_SWIZZLE_64B);
  if (!rc) rc = make_map_2d(&mb, g.split, split_rows, g.nb, 4, BK, BNH, CU_TENSOR_MAP_SWIZZLE_64B);
  const int64_t c_rows = g.noff() > 0 ? g.noff() * g.nb : 32;
  if (!rc) rc = make_map_2d(&mc, g.sp, c_rows, g.nb, 4, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  WorkW w;
  w.slot0 = s0;
  w.nsubm = g.nb / (2 * BM);
  w.nitems = (int)(scnt * w.nsubm);
  w.span = span;
  w.l2pf = mt_opt_wide_l2pf();
  int dev = 0;
  cudaGetDevice(&dev);
  if (!g_smw) cudaDeviceGetAttribute(&g_smw, cudaDevAttrMultiProcessorCount, dev);
  static int* counters[64] = {nullptr};
  static unsigned next_counter[64] = {0};
  if (dev < 0 || dev >= 64) { mt_set_error("device index out of range"); return MT_E_CUDA; }
  if (!counters[dev] && mt_cuda_check(cudaMalloc(&counters[dev], 2 * 256 * sizeof(int)), "counter alloc"))
    return MT_E_CUDA;
  w.counter = counters[dev] + 2 * (next_counter[dev]++ % 256);
  if (mt_cuda_check(cudaMemsetAsync(w.counter, 0, 2 * sizeof(int), st), "counter reset"))
    return MT_E_CUDA;
  int pairs = (ctas > 0 ? ctas : g_smw) / 2;
  if (pairs > w.nitems) pairs = w.nitems;
  if (pairs < 1) pairs = 1;
  cudaFuncSetAttribute(tc2w_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  tc2w_update_kernel<<<2 * pairs, NUM_THREADS, SMEM_BYTES, st>>>(g, k, w, ma, mb, mc);
  MT_LAUNCH_CHECK("tc2w_update_kernel");
  return MT_OK;
}
