// FP32-accurate 3xTF32 on CTA pairs: the off-band trailing update, the
// panel-column update and the off-band panel TRSM with the TMEM accumulator
// FLUSHED into a round-to-nearest FP32 running sum in registers every KC
// K-slabs.
//
//   C_ij <- C_ij - A_ik A_jk^T      (kernels.gemm FP32 path, factor.py:273-274)
//   X_ik  = B_ik W^T, W = L_kk^-1   (kernels.trsm FP32 path, factor.py:264)
//
// Why: tcgen05.mma adds every K=8 partial product into the FP32 TMEM
// accumulator with round-toward-zero.  Over a 512-deep update that is 192
// biased roundings at the magnitude of the running sum -- a systematic error
// FP32 FFMA / OpenBLAS sgemm (round-to-nearest) does not have
// (tools/emulate_tf32x3.py, tools/emulate_flush.py).  The bias of a chunk
// grows with its length, so each accumulation restarts from zero every 32
// K-columns (KC slabs; 4 MMA k-steps) and the epilogue adds the chunk into
// its registers with ordinary round-to-nearest FADDs; C_new = RN(C - sum).
// CPU emulation of exactly this arithmetic puts kriging within 1.3x of the
// reference's sgemm deviation from DP (RZ unflushed: 12.6x).
//
// Layout (one CTA per SM, cluster (2,1,1), 320 threads):
//   warp 0  TMA producer (+ the leader's dynamic work queue, as tc2_update.cu)
//   warp 1  leader: tcgen05.mma.cta_group::2 issuer, M = 256, N = 256; the two
//           TMEM buffers (256 columns each) alternate per K chunk, not per item
//   warps 2..9  epilogue: two warps per TMEM lane quadrant, 128 columns each;
//           128 running-sum registers per thread (lane = accumulator row).
//           Per chunk: 4 tcgen05.ld 32x32b.x32 + FADDs (TMEM reads measured at
//           ~26 B/clk per warp on B200, tools/tmem_bw.cu: 8 warps drain a
//           128 KB chunk in ~0.6 us of the chunk's ~0.8 us of MMA).
//           Item end: C streamed through 3 SWIZZLE_128B 32x32 chunk slots per
//           warp with TMA (loaded during the item), result stored by TMA; the
//           panel-column update and the TRSM also store the TF32 hi/lo split
//           of their outputs (operands of the next step) by TMA.
// Deterministic: every output element gets the same MMA and FADD sequence in
// the same order from exactly one pair, whatever the schedule.
#include <cuda.h>

#include "tma.cuh"
#include "tc2_common.cuh"

namespace {
using namespace mt_tma;
using namespace mt_pair;

constexpr int BM = 128;   // accumulator rows per CTA (pair M = 256)
constexpr int BN = 256;   // pair N (one MMA)
constexpr int BNH = 128;  // rows of B each CTA stages
#ifndef MT_TCF_BK
#define MT_TCF_BK 32
#endif
// K columns per operand slab: 32 (128-byte rows, SWIZZLE_128B; default) or
// 16 (64-byte rows, SWIZZLE_64B).  The wider slab halves the TMA row requests
// per byte.  Same-box A/B at N=262144 (bitwise-identical results,
// profiles/ab_tcf_stages_r02.txt): 16-column slabs x 4 stages + 3 C slots of
// 32 columns 40.10 s; 32 x 2 + 3 x 32 38.99 s; 32 x 3 + 2 C slots of 16
// columns 37.81 s (default)
constexpr int BK = MT_TCF_BK;
static_assert(BK == 16 || BK == 32, "slab width");
constexpr CUtensorMapSwizzle kSwz = BK == 16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
#ifndef MT_TCF_KC
#define MT_TCF_KC (32 / MT_TCF_BK)
#endif
constexpr int KC = MT_TCF_KC;  // K slabs per TMEM chunk
static_assert((256 / MT_TCF_BK) % KC == 0, "KC must divide the item's slab granularity");
// (KC * BK = 32: the accumulator restarts every 32 K-columns at either slab width)
#ifndef MT_TCF_STAGES
#define MT_TCF_STAGES (MT_TCF_BK == 32 ? 3 : 4)
#endif
constexpr int STAGES = MT_TCF_STAGES;
constexpr int A_BYTES = BM * BK * 4;                  // 8 KB
constexpr int B_BYTES = BNH * BK * 4;                 // 8 KB
constexpr int STAGE_BYTES = 2 * (A_BYTES + B_BYTES);  // hi + lo = 32 KB
#ifndef MT_TCF_EPI
#define MT_TCF_EPI 8
#endif
constexpr int EPI_WARPS = MT_TCF_EPI;  // 8 or 16: 2 or 4 warps per TMEM lane quadrant
static_assert(EPI_WARPS == 8 || EPI_WARPS == 16, "epilogue warps");
constexpr int COLS_W = BN / (EPI_WARPS / 4);  // columns per epilogue warp
#ifndef MT_TCF_RED_PREFETCH
// reduce-add epilogue: 1 = prefetch the item's C into L2 at its start.  Off by
// default: the reduce-adds are fire-and-forget, so C latency never stalls the
// warp, and the early prefetch only competed for L2 with the operand slabs
// (no prefetch: 1.1% faster at N=262144, DRAM 112.9 -> 111.8 GB per launch)
#define MT_TCF_RED_PREFETCH 0
#endif
#ifndef MT_TCF_L2HINT
#define MT_TCF_L2HINT 0  // 1 = B slabs evict_last, C reduce-adds evict_first (A/B)
#endif
#ifndef MT_TCF_LDX
#define MT_TCF_LDX 16
#endif
constexpr int LDX = MT_TCF_LDX;  // TMEM columns per tcgen05.ld (+ wait::ld) in the drain
static_assert(LDX == 16 || LDX == 32, "TMEM load width");
constexpr int NUM_THREADS = 64 + 32 * EPI_WARPS;
#ifndef MT_TCF_CSLOTS
#define MT_TCF_CSLOTS (MT_TCF_BK == 32 ? 2 : 3)
#endif
#ifndef MT_TCF_CW
#define MT_TCF_CW (MT_TCF_BK == 32 ? 16 : 32)
#endif
// C chunks: 32 rows x CW columns (CW = 32: 128-byte rows, SWIZZLE_128B; 16:
// 64-byte rows, SWIZZLE_64B); CSLOTS per epilogue warp (2 or 3)
constexpr int CW = MT_TCF_CW, NE = CW / 4;  // NE: 16-byte groups per chunk row
static_assert(CW == 32 || CW == 16 || CW == 8, "C chunk width");
constexpr int NCW = COLS_W / CW;  // C chunks per warp and item
constexpr CUtensorMapSwizzle kSwzC = CW == 32 ? CU_TENSOR_MAP_SWIZZLE_128B
                                    : (CW == 16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
constexpr int CSLOTS = MT_TCF_CSLOTS, CSLOT_BYTES = 32 * CW * 4;
static_assert(CSLOTS >= 2 && CSLOTS <= 4, "C-chunk slots");
constexpr int EPI_BYTES = EPI_WARPS * CSLOTS * CSLOT_BYTES;  // 96 KB at 3 slots
constexpr int TMEM_COLS = 512;                               // 2 chunk buffers x 256 columns
constexpr int SCHED = 4;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 768;
static_assert(SMEM_BYTES <= 232448, "shared memory");

// kind::tf32, D f32, A/B tf32 K-major, N = 256, M = 256 (cta_group::2)
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(256 >> 4) << 24);

// K-major UMMA smem descriptor of a swizzled operand slab: 8-row groups of
// BK*4 bytes (SBO), layout SWIZZLE_64B (4) or SWIZZLE_128B (2)
__device__ __forceinline__ uint64_t opdesc(const void* p) {
  const uint64_t a = (smem_u32(p) >> 4) & 0x3FFF;
  return a | ((uint64_t)((8 * BK * 4) >> 4) << 32) | (1ull << 46) |
         ((uint64_t)(BK == 16 ? 4 : 2) << 61);
}
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void ld32(uint32_t (&v)[32], uint32_t taddr) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
        "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
        "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// physical 16-byte group of group e in row `row` of a swizzled C chunk
// (16-byte-group index XOR address bits 7..9 for 128 B rows, 7..8 for 64 B
// rows, 7 for 32 B rows)
__device__ __forceinline__ int swz(int e, int row) {
  return CW == 32 ? (e ^ (row & 7)) : (CW == 16 ? (e ^ ((row >> 1) & 3)) : (e ^ ((row >> 2) & 1)));
}
__device__ __forceinline__ void ld16(uint32_t (&v)[16], uint32_t taddr) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void ldtm(uint32_t (&v)[16], uint32_t taddr) { ld16(v, taddr); }
__device__ __forceinline__ void ldtm(uint32_t (&v)[32], uint32_t taddr) { ld32(v, taddr); }
// 2-CTA TMA multicast (cta_group::2): the box lands at the same smem offset in
// every CTA of `mask`; each destination's bytes complete on the `full` barrier
// of that destination's pair leader (the peer bit of the barrier address
// cleared, as CUTLASS's SM100_TMA_2SM_LOAD_MULTICAST)
__device__ __forceinline__ void tma_load_pair_mc(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                 uint16_t mask, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%4, %5}], [%2], %3;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar) & 0xFEFFFFFFu), "h"(mask), "r"(c0), "r"(c1)
      : "memory");
}
// MMA completion arriving once on the barrier at this offset in every CTA of mask
__device__ __forceinline__ void umma2_commit_mask(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void prefetch_l2_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"((uint64_t)map),
               "r"(c0), "r"(c1)
               : "memory");
}

struct WorkF {
  int64_t slot0;
  int nitems;  // slots * nsubm * nsubn (pair items of 256 x 256)
  int nsubm, nsubn;
  int* counter;  // [work queue head, pairs started]
  int presplit;  // the column-(k+1) update also writes its outputs' TF32 split
  unsigned long long* span;
  int mlo, mhi, sw;  // update: owned column range, super-column width (0 = slot order)
  int stats;         // option 16: accumulate MMA-issuer wait cycles
  int red;           // option 17: C -= sum as a TMA reduce-add of -sum (no C load)
};

enum { OUT_UPDATE = 0, OUT_PRESPLIT = 1, OUT_TRSM = 2 };

// diagnostics (option 16): MMA-issuer cycles spent waiting for operands
// (full), for a drained TMEM chunk buffer (tempty) and in total, summed over
// the pair leaders of every launch since the last mt_tcf_stats() read
__device__ unsigned long long g_tcf_stats[4];

// CL = CTAs per cluster: 2 (one pair, 256 x 256 items) or 4 (two pairs on
// 512 x 256 items sharing the B operand: each CTA loads its 128 rows of A and
// multicasts half of its pair-half of B to the CTA of the same pair rank in
// the other pair -- 24 instead of 32 KB of L2->SM operand traffic per slab)
template <bool TRSM, int CL>
__device__ __forceinline__ void tcf_body(const Grid& g, int k, const WorkF& w,
                                         const CUtensorMap& map_a, const CUtensorMap& map_b,
                                         const CUtensorMap& map_c, const CUtensorMap& map_s) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* epi = smem + STAGES * STAGE_BYTES;
  uint64_t* full = (uint64_t*)(epi + EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;
  uint64_t* sempty = sfull + SCHED;
  uint64_t* cbar = sempty + SCHED;  // EPI_WARPS * CSLOTS C-chunk load barriers
  int* sitem = (int*)(cbar + EPI_WARPS * CSLOTS);
  int* si = sitem + SCHED;
  int* sj = si + SCHED;
  uint32_t* tmem_slot = (uint32_t*)(sj + SCHED);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // co-scheduled band update
  const uint32_t rank = cta_rank();
  const uint32_t prank = rank & 1;          // rank inside the pair
  const uint32_t plead = rank & ~1u;        // the pair's leader (MMA issuer, TMEM owner of record)
  const bool leader = prank == 0;           // pair leader
  const bool qowner = rank == 0;            // owner of the cluster's work queue
  const uint16_t pair_mask = (uint16_t)(3u << plead);
  const int nb = g.nb;
  const int nsub = w.nsubm * w.nsubn;
  auto item_ksteps = [&](int item) {
    return TRSM ? ((item % nsub) % w.nsubn + 1) * (BN / BK) : nb / BK;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL / 2);  // one commit per pair (CL = 4: B is shared by both pairs)
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * EPI_WARPS);  // leader: local + peer epilogue warps
    }
    for (int s = 0; s < SCHED; ++s) {
      mbar_init(&sfull[s], 1);
      // queue owner: MMA issuers + epilogue warps of every CTA + peer producers
      mbar_init(&sempty[s], CL / 2 + CL * EPI_WARPS + CL - 1);
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
      if (qowner) mbar_arrive_relaxed(&sempty[s]);
      else mbar_arrive_cl_relaxed(peer_addr(&sempty[s], 0));
    }
    return item;
  };

  if (warp == 0) {
    // ------------------------------------------------ work queue + TMA producer
    if (lane == 0) {
      if (qowner && !TRSM && g.yield) atomicAdd(w.counter + 1, 1);  // clusters started
      const int nclusters = (int)(gridDim.x / CL);
      uint32_t it = 0;
      for (uint32_t li = 0;; ++li) {
        const int s = li % SCHED;
        int item, i = 0, j = 0;
        if (qowner) {
          mbar_wait(&sempty[s], ((li / SCHED) & 1) ^ 1);
          if (g.failed()) {
            item = -1;
          } else if (!TRSM && g.yield && *(volatile int*)g.yield > 0 &&
                     *(volatile int*)(w.counter + 1) < nclusters && atomicSub(g.yield, CL) > 0) {
            item = -1;  // SM-yield request (see tc2_update.cu)
          } else {
            item = atomicAdd(w.counter, 1);
            if (item >= w.nitems) item = -1;
          }
          if (item >= 0) {
            if (!TRSM && w.sw > 0) super_tile_ij(g, item / nsub, w.mlo, w.mhi, w.sw, i, j);
            else g.off_slot_ij(w.slot0 + item / nsub, i, j);
          }
          sitem[s] = item; si[s] = i; sj[s] = j;
#pragma unroll
          for (uint32_t r = 1; r < CL; ++r) {
            st_cl_u32(peer_addr(&sitem[s], r), (uint32_t)item);
            st_cl_u32(peer_addr(&si[s], r), (uint32_t)i);
            st_cl_u32(peer_addr(&sj[s], r), (uint32_t)j);
          }
          mbar_arrive(&sfull[s]);
#pragma unroll
          for (uint32_t r = 1; r < CL; ++r) mbar_arrive_cl(peer_addr(&sfull[s], r));
        } else {
          mbar_wait_cl(&sfull[s], (li / SCHED) & 1);
          item = *(volatile int*)&sitem[s];
          i = *(volatile int*)&si[s];
          j = *(volatile int*)&sj[s];
          if ((item ^ i ^ j) != 0x7fffffff) mbar_arrive_cl_relaxed(peer_addr(&sempty[s], 0));
        }
        if (item < 0) break;
        const int sub = item % nsub;
        const int m0 = (sub / w.nsubn) * (CL * BM) + (int)rank * BM;
        // CL = 4: this CTA loads rows [pair * 64, +64) of its 128-row half of B
        // and multicasts them to the CTA of the same pair rank in both pairs
        const int n0 = (sub % w.nsubn) * BN + (int)prank * BNH + (CL == 4 ? (int)(rank >> 1) * 64 : 0);
        const int arow = TRSM ? (int)g.presplit_row(i) + m0 : (int)g.split_row(i, k) + m0;
        const int brow = TRSM ? (int)g.winv_row() + n0 : (int)g.split_row(j, k) + n0;
        const uint16_t bmask = (uint16_t)(0x5u << prank);  // CTAs {prank, prank + 2}
        const int boff = CL == 4 ? (int)(rank >> 1) * 64 * BK * 4 : 0;
        const int ksteps = item_ksteps(item);
        for (int ks = 0; ks < ksteps; ++ks, ++it) {
          const int st = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty[st], ph ^ 1);
          unsigned char* sb = smem + st * STAGE_BYTES;
          if (leader) mbar_expect_tx(&full[st], 2 * STAGE_BYTES);
          const uint32_t bar = peer_addr(&full[st], plead);
          tma_load_pair(sb, &map_a, bar, ks * BK, arow);                               // A hi
          tma_load_pair(sb + A_BYTES + B_BYTES, &map_a, bar, ks * BK, arow + nb);      // A lo
          if constexpr (CL == 4) {
            tma_load_pair_mc(sb + A_BYTES + boff, &map_b, &full[st], bmask, ks * BK, brow);
            tma_load_pair_mc(sb + 2 * A_BYTES + B_BYTES + boff, &map_b, &full[st], bmask, ks * BK,
                             brow + nb);
          } else if (MT_TCF_L2HINT && !TRSM) {
            // column operands stay in L2 for the whole super-column
            const uint64_t pol = l2_policy_evict_last();
            tma_load_pair_hint(sb + A_BYTES, &map_b, bar, ks * BK, brow, pol);
            tma_load_pair_hint(sb + 2 * A_BYTES + B_BYTES, &map_b, bar, ks * BK, brow + nb, pol);
          } else {
            tma_load_pair(sb + A_BYTES, &map_b, bar, ks * BK, brow);                     // B hi
            tma_load_pair(sb + 2 * A_BYTES + B_BYTES, &map_b, bar, ks * BK, brow + nb);  // B lo
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (leader only)
    if (leader) {
      uint32_t it = 0, ch = 0;
      const bool stats = w.stats;
      unsigned long long w_full = 0, w_tempty = 0;
      const unsigned long long t_start = stats ? clock64() : 0;
      for (uint32_t li = 0;; ++li) {
        const int item = next_item(li, nullptr, nullptr);
        if (item < 0) break;
        const int ksteps = item_ksteps(item);
        for (int ks = 0; ks < ksteps; ++ks, ++it) {
          const uint32_t b = ch & 1;
          const bool c_first = (ks % KC) == 0, c_last = (ks % KC) == KC - 1;
          if (c_first) {
            const unsigned long long t0 = stats ? clock64() : 0;
            mbar_wait_cl(&tempty[b], ((ch >> 1) & 1) ^ 1);  // chunk buffer drained
            if (stats) w_tempty += clock64() - t0;
            asm volatile("tcgen05.fence::after_thread_sync;");
          }
          const int s = it % STAGES;
          const unsigned long long t1 = stats ? clock64() : 0;
          mbar_wait(&full[s], (it / STAGES) & 1);
          if (stats) w_full += clock64() - t1;
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (lane == 0) {
            unsigned char* st = smem + s * STAGE_BYTES;
            const unsigned char* ahi = st;
            const unsigned char* bhi = st + A_BYTES;
            const unsigned char* alo = st + A_BYTES + B_BYTES;
            const unsigned char* blo = alo + A_BYTES;
            const uint32_t dcol = tmem_base + b * BN;
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const int off = kk * 32;
              umma(dcol, opdesc(alo + off), opdesc(bhi + off), (c_first && kk == 0) ? 0u : 1u);
              umma(dcol, opdesc(ahi + off), opdesc(blo + off), 1u);
              umma(dcol, opdesc(ahi + off), opdesc(bhi + off), 1u);
            }
            // stage s is free in every CTA that received part of it: both pairs
            // when B was multicast (each CTA's empty[s] then counts 2 commits)
            umma2_commit_mask(&empty[s], CL == 4 ? (uint16_t)0xF : pair_mask);
            if (c_last) umma2_commit_mask(&tfull[b], pair_mask);
          }
          __syncwarp();
          if (c_last) ++ch;
        }
      }
      if (stats && lane == 0) {
        atomicAdd(&g_tcf_stats[0], w_full);
        atomicAdd(&g_tcf_stats[1], w_tempty);
        atomicAdd(&g_tcf_stats[2], clock64() - t_start);
        atomicAdd(&g_tcf_stats[3], 1ull);
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2..9, both CTAs)
    const int ew = warp - 2;
    const int q = warp & 3;     // TMEM lane quadrant this warp may access
    const int half = ew >> 2;   // column part of the item (COLS_W wide)
    unsigned char* slots = epi + ew * CSLOTS * CSLOT_BYTES;
    uint64_t* wbar = cbar + ew * CSLOTS;
    const uint32_t tempty_l0 = peer_addr(&tempty[0], plead), tempty_l1 = peer_addr(&tempty[1], plead);
    uint32_t phb = 0;  // bit s: parity of slot s's next C load
    uint32_t ch = 0;
    auto load_c = [&](int s, int col, int row) {  // lane 0; slot s must be free
      mbar_expect_tx(&wbar[s], CSLOT_BYTES);
      tma_load_2d(slots + s * CSLOT_BYTES, &map_c, &wbar[s], col, row);
    };
    auto wait_c = [&](int s) {
      mbar_wait(&wbar[s], (phb >> s) & 1);
      phb ^= 1u << s;
    };
    for (uint32_t li = 0;; ++li) {
      int i, j;
      const int item = next_item(li, &i, &j);
      if (item < 0) break;
      const int sub = item % nsub;
      const int row0 = (sub / w.nsubn) * (CL * BM) + (int)rank * BM + q * 32;  // row in the tile
      const int n0 = (sub % w.nsubn) * BN + half * COLS_W;                    // first column
      const int out = TRSM ? OUT_TRSM : ((w.presplit && j == k + 1) ? OUT_PRESPLIT : OUT_UPDATE);
      // TMA rows: output tile (i, j) (TRSM: j == k) in the off-band pool, and
      // the split buffer rows of its TF32 hi part (lo = + nb)
      const int crow = (int)(g.sslot(i, j) * nb) + row0;
      const int srow = out == OUT_TRSM ? (int)g.split_row(i, k) + row0
                                       : (int)g.presplit_row(i) + row0;
      const int nch = item_ksteps(item) / KC;
      float sum[COLS_W];
#pragma unroll
      for (int u = 0; u < COLS_W; ++u) sum[u] = 0.f;
      const uint32_t tq = tmem_base + ((uint32_t)(q * 32) << 16) + half * COLS_W;
#pragma unroll 1
      for (int c = 0; c < nch; ++c) {
        const uint32_t b = ch & 1;
        mbar_wait(&tfull[b], (ch >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int m = 0; m < COLS_W / LDX; ++m) {
          uint32_t v[LDX];
          ldtm(v, tq + b * BN + m * LDX);
#pragma unroll
          for (int u = 0; u < LDX; ++u) sum[LDX * m + u] += __uint_as_float(v[u]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive_cl_relaxed(b ? tempty_l1 : tempty_l0);
        ++ch;
        if (c == 0 && out != OUT_TRSM && lane == 0) {
          // C of this item: slots free once the previous item's stores were read
          if (out == OUT_UPDATE && w.red) {
            if (MT_TCF_RED_PREFETCH)
              for (int m = 0; m < NCW; ++m) prefetch_l2_2d(&map_c, n0 + m * CW, crow);
          } else if (out == OUT_UPDATE) {
            bulk_wait_read<0>();
            for (int m = 0; m < CSLOTS; ++m) load_c(m, n0 + m * CW, crow);
            for (int m = CSLOTS; m < NCW; ++m) prefetch_l2_2d(&map_c, n0 + m * CW, crow);
          } else {
            bulk_wait_read<0>();
            load_c(0, n0, crow);
            for (int m = 1; m < NCW; ++m) prefetch_l2_2d(&map_c, n0 + m * CW, crow);
          }
        }
      }
      // ---- output: lane = row, CW columns per chunk m, swizzled slots
      // x[0..CW-1] -> slot s row `lane`: the values (part 0), or their TF32 hi (1) / lo (2)
      auto put = [&](int s, const float* x, int part) {
        const uint32_t rowa = smem_u32(slots + s * CSLOT_BYTES) + lane * (CW * 4);
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          float y[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            float h, l;
            mt_tf32_split(x[4 * e + u], h, l);
            y[u] = part == 0 ? x[4 * e + u] : (part == 1 ? h : l);
          }
          sts128(rowa + (swz(e, lane) << 4), make_float4(y[0], y[1], y[2], y[3]));
        }
      };
      if (out == OUT_UPDATE && w.red) {
        // C - sum == C + (-sum) in IEEE arithmetic: the TMA unit adds -sum into
        // C at L2, the warp only waits for a slot's previous reduce to have
        // read its source (chunk 0: every earlier bulk op of this warp, which
        // may have used the slots in another pattern)
#pragma unroll
        for (int m = 0; m < NCW; ++m) {
          const int s = m % CSLOTS;
          if (lane == 0) {
            if (m == 0) bulk_wait_read<0>();
            else bulk_wait_read<CSLOTS - 1>();
          }
          __syncwarp();
          const uint32_t rowa = smem_u32(slots + s * CSLOT_BYTES) + lane * (CW * 4);
#pragma unroll
          for (int e = 0; e < NE; ++e)
            sts128(rowa + (swz(e, lane) << 4),
                   make_float4(-sum[CW * m + 4 * e], -sum[CW * m + 4 * e + 1],
                               -sum[CW * m + 4 * e + 2], -sum[CW * m + 4 * e + 3]));
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            if (MT_TCF_L2HINT)  // C is not read again in this step
              tma_reduce_add_2d_hint(&map_c, slots + s * CSLOT_BYTES, n0 + m * CW, crow,
                                     l2_policy_evict_first());
            else
              tma_reduce_add_2d(&map_c, slots + s * CSLOT_BYTES, n0 + m * CW, crow);
            bulk_commit();
          }
        }
      } else if (out == OUT_UPDATE) {
#pragma unroll
        for (int m = 0; m < NCW; ++m) {
          const int s = m % CSLOTS;
          wait_c(s);
          const uint32_t rowa = smem_u32(slots + s * CSLOT_BYTES) + lane * (CW * 4);
#pragma unroll
          for (int e = 0; e < NE; ++e) {
            const uint32_t a = rowa + (swz(e, lane) << 4);
            float4 cc = lds128(a);
            cc.x -= sum[CW * m + 4 * e];
            cc.y -= sum[CW * m + 4 * e + 1];
            cc.z -= sum[CW * m + 4 * e + 2];
            cc.w -= sum[CW * m + 4 * e + 3];
            sts128(a, cc);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&map_c, slots + s * CSLOT_BYTES, n0 + m * CW, crow);
            bulk_commit();
            if (m + CSLOTS < NCW) {  // chunk m + CSLOTS reuses this slot (L2-prefetched)
              bulk_wait_read<0>();
              load_c(s, n0 + (m + CSLOTS) * CW, crow);
            }
          }
        }
      } else {
#pragma unroll
        for (int m = 0; m < NCW; ++m) {
          float x[CW];
          if (out == OUT_PRESPLIT) {
            wait_c(0);
            const uint32_t rowa = smem_u32(slots) + lane * (CW * 4);
#pragma unroll
            for (int e = 0; e < NE; ++e) {
              const float4 cc = lds128(rowa + (swz(e, lane) << 4));
              x[4 * e] = cc.x - sum[CW * m + 4 * e];
              x[4 * e + 1] = cc.y - sum[CW * m + 4 * e + 1];
              x[4 * e + 2] = cc.z - sum[CW * m + 4 * e + 2];
              x[4 * e + 3] = cc.w - sum[CW * m + 4 * e + 3];
            }
          } else {
            if (lane == 0) bulk_wait_read<0>();  // slots free (previous chunk's stores read)
            __syncwarp();
#pragma unroll
            for (int u = 0; u < CW; ++u) x[u] = sum[CW * m + u];
          }
          put(0, x, 0);
          put(1, x, 1);
          if (CSLOTS > 2) put(2, x, 2);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&map_c, slots, n0 + m * CW, crow);
            tma_store_2d(&map_s, slots + CSLOT_BYTES, n0 + m * CW, srow);
            if (CSLOTS > 2) tma_store_2d(&map_s, slots + 2 * CSLOT_BYTES, n0 + m * CW, srow + nb);
            bulk_commit();
          }
          if (CSLOTS == 2) {  // the TF32 lo part goes through slot 1 once hi was read
            if (lane == 0) bulk_wait_read<0>();
            __syncwarp();
            put(1, x, 2);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&map_s, slots + CSLOT_BYTES, n0 + m * CW, srow + nb);
              bulk_commit();
            }
          }
          if (lane == 0) {
            if (out == OUT_PRESPLIT && m < NCW - 1) {
              bulk_wait_read<0>();
              load_c(0, n0 + (m + 1) * CW, crow);
            }
          }
          __syncwarp();
        }
      }
    }
    if (lane == 0) bulk_wait_all();  // stores complete before the kernel ends
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

template <int CL>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    tcf_update_kernel(Grid g, int k, WorkF w, const __grid_constant__ CUtensorMap map_a,
                      const __grid_constant__ CUtensorMap map_b,
                      const __grid_constant__ CUtensorMap map_c,
                      const __grid_constant__ CUtensorMap map_s) {
  tcf_body<false, CL>(g, k, w, map_a, map_b, map_c, map_s);
}

template <int CL>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    tcf_trsm_kernel(Grid g, int k, WorkF w, const __grid_constant__ CUtensorMap map_a,
                    const __grid_constant__ CUtensorMap map_b,
                    const __grid_constant__ CUtensorMap map_c,
                    const __grid_constant__ CUtensorMap map_s) {
  tcf_body<true, CL>(g, k, w, map_a, map_b, map_c, map_s);
}

template <int CL>
int launch_tcf(bool trsm, int clusters, cudaStream_t st, const Grid& g, int k, const WorkF& w,
               const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc,
               const CUtensorMap& ms) {
  auto kern = trsm ? tcf_trsm_kernel<CL> : tcf_update_kernel<CL>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL * clusters);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (mt_cuda_check(cudaLaunchKernelEx(&cfg, kern, g, k, w, ma, mb, mc, ms),
                    trsm ? "tcf_trsm_kernel" : "tcf_update_kernel"))
    return MT_E_CUDA;
  return MT_OK;
}

int g_smf = 0;

}  // namespace

// launch over the off-band slot range [s0, s0 + scnt) of step k (update) or
// panel k (trsm); `ctas` caps the grid (rounded down to pairs)
int mt_tcf_launch(const Grid& g, int k, int64_t s0, int64_t scnt, int ctas, bool trsm, int presplit,
                  cudaStream_t st, unsigned long long* span, int jlo, int jhi) {
  if (scnt <= 0) return MT_OK;
  // 4-CTA clusters (two pairs sharing B by multicast) need 512-row items
  const int CL = (mt_opt_tcf_cluster4() && g.nb % (4 * BM) == 0) ? 4 : 2;
  CUtensorMap ma, mb, mc, ms;
  const int64_t split_rows = g.split_rows();
  int rc = make_map_2d(&ma, g.split, split_rows, g.nb, 4, BK, BM, kSwz);
  if (!rc) rc = make_map_2d(&mb, g.split, split_rows, g.nb, 4, BK, CL == 4 ? BNH / 2 : BNH, kSwz);
  const int64_t c_rows = g.noff() > 0 ? g.noff() * g.nb : 32;
  if (!rc) rc = make_map_2d(&mc, g.sp ? (const void*)g.sp : (const void*)g.split, c_rows, g.nb, 4, CW,
                            32, kSwzC);
  if (!rc) rc = make_map_2d(&ms, g.split, split_rows, g.nb, 4, CW, 32, kSwzC);
  if (rc) return rc;
  WorkF w;
  w.slot0 = s0;
  w.nsubm = g.nb / (CL * BM);
  w.nsubn = g.nb / BN;
  w.nitems = (int)(scnt * w.nsubm * w.nsubn);
  w.presplit = presplit;
  w.span = span;
  w.mlo = g.owned_before(jlo);
  w.mhi = g.owned_before(jhi);
  w.sw = (!trsm && jhi > jlo + 1 && g.rs == 1) ? mt_opt_super_cols() : 0;
  w.stats = mt_opt_tcf_stats();
  w.red = mt_opt_tcf_reduce();
  int dev = 0;
  cudaGetDevice(&dev);
  if (!g_smf) cudaDeviceGetAttribute(&g_smf, cudaDevAttrMultiProcessorCount, dev);
  static int* counters[64] = {nullptr};
  static unsigned next_counter[64] = {0};
  if (dev < 0 || dev >= 64) { mt_set_error("device index out of range"); return MT_E_CUDA; }
  if (!counters[dev] && mt_cuda_check(cudaMalloc(&counters[dev], 2 * 256 * sizeof(int)), "counter alloc"))
    return MT_E_CUDA;
  w.counter = counters[dev] + 2 * (next_counter[dev]++ % 256);
  if (mt_cuda_check(cudaMemsetAsync(w.counter, 0, 2 * sizeof(int), st), "counter reset"))
    return MT_E_CUDA;
  int clusters = (ctas > 0 ? ctas : g_smf) / CL;
  if (!trsm && g.yield && ctas <= 0) clusters = 2 * g_smf / CL;  // oversubscribed: refills yielded SMs
  if (clusters > w.nitems) clusters = w.nitems;
  if (clusters < 1) clusters = 1;
  return CL == 4 ? launch_tcf<4>(trsm, clusters, st, g, k, w, ma, mb, mc, ms)
                 : launch_tcf<2>(trsm, clusters, st, g, k, w, ma, mb, mc, ms);
}

// option-16 diagnostics: {cycles waiting for operands, for TMEM, total, issuers}
extern "C" int mt_tcf_stats(double* out4) {
  unsigned long long h[4] = {0, 0, 0, 0};
  if (mt_cuda_check(cudaMemcpyFromSymbol(h, g_tcf_stats, sizeof(h)), "tcf stats")) return MT_E_CUDA;
  const unsigned long long z[4] = {0, 0, 0, 0};
  if (mt_cuda_check(cudaMemcpyToSymbol(g_tcf_stats, z, sizeof(z)), "tcf stats reset")) return MT_E_CUDA;
  for (int q = 0; q < 4; ++q) out4[q] = (double)h[q];
  return MT_OK;
}
