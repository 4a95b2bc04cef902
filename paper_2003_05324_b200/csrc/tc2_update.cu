// FP32 (off-band) trailing update and off-band panel TRSM on CTA PAIRS:
// tcgen05.mma.cta_group::2, 3xTF32 (same arithmetic as tc_update.cu).
//
//   C_ij <- C_ij - A_ik A_jk^T      (kernels.gemm FP32 path, factor.py:273-274)
//   X_ik  = B_ik W^T, W = L_kk^-1   (kernels.trsm FP32 path, factor.py:264)
//
// Why pairs: the single-CTA kernel (M=128, N=256) stages 48 KB of TF32 hi/lo
// operands per 16-wide K slab through TMA, i.e. 64 B/clk/SM at full MMA rate,
// above what L2->SM delivers (~42 B/clk/SM chip-wide, B300_MICROARCH "TMA
// chip-throughput"); ncu showed the tensor pipe ~68% busy with the MMA issuer
// waiting on operands.  A CTA pair computes a 256 x 256 block with one
// M=256 UMMA: each CTA stages its own 128 rows of A and HALF of B (128 rows),
// 32 KB per slab for the same MMA time -- 1.5x less operand traffic per flop.
//
// Roles (192 threads per CTA, one CTA per SM, cluster (2,1,1)):
//   warp 0  TMA producer in both CTAs; the leader (rank 0) also owns the
//           dynamic work queue and forwards each item to the peer through
//           distributed shared memory.  Both CTAs' TMA loads complete on the
//           leader's `full` barrier (cta_group::2 TMA).
//   warp 1  leader: single-thread tcgen05.mma.cta_group::2 issuer; its commits
//           multicast to both CTAs' `empty` / `tfull` barriers.  Both CTAs'
//           warp 1 allocate / free TMEM (cta_group::2).
//   warps 2-5  epilogue of the CTA's own 128 accumulator rows (TMEM lanes),
//           as in tc_update.cu; they release the accumulator on the leader's
//           `tempty` (4 local + 4 remote arrivals).
// Every output element is produced by one pair per step with the same MMA
// sequence (K slabs in order, lo*hi, hi*lo, hi*hi) as in the single-CTA
// kernel: deterministic, schedule-invariant, and bit-identical to it
// (tests/test_gpu_tc.py::test_cta_pair_kernel_bitwise_equals_single_cta).
#include <cuda.h>

#include "tma.cuh"

namespace {
using namespace mt_tma;

constexpr int BM = 128;               // accumulator rows per CTA (pair M = 256)
#ifndef MT_TC2_SPLITACC
#define MT_TC2_SPLITACC 0
#endif
// MT_TC2_SPLITACC: accumulate the hi*hi products and the two correction
// products (lo*hi, hi*lo) in separate TMEM accumulators, summed in FP32 by the
// epilogue.  The tensor core adds each K=8 partial into TMEM with
// round-toward-zero; keeping the small correction terms out of the large
// accumulator removes 2/3 of those biased additions at full magnitude
// (tools/emulate_tf32x3.py).  Costs N = 128 items (TMEM holds 2 x 2 x 128).
constexpr int BN = MT_TC2_SPLITACC ? 128 : 256;  // pair N; each CTA stages BN / 2 rows of B
constexpr int ACC_STRIDE = MT_TC2_SPLITACC ? 2 * BN : BN;  // TMEM columns per accumulator buffer
constexpr int BNH = BN / 2;
#ifndef MT_TC2_TMAEPI
#define MT_TC2_TMAEPI 1
#endif
// MT_TC2_TMAEPI: the bulk update's epilogue streams C through shared memory
// with TMA (4 x 4 KB SWIZZLE_128B chunk slots per warp, loads issued up to 3
// chunks ahead, results stored back by TMA); 5 operand stages leave room for it
constexpr int BK = 16, STAGES = MT_TC2_SPLITACC ? 6 : (MT_TC2_TMAEPI ? 5 : 6);
constexpr int A_BYTES = BM * BK * 4;  // 8 KB
constexpr int B_BYTES = BNH * BK * 4; // 8 KB (4 KB with split accumulators)
constexpr int STAGE_BYTES = 2 * (A_BYTES + B_BYTES);  // hi + lo = 32 KB (24 KB split)
#ifndef MT_TC2_EPI
#define MT_TC2_EPI 4
#endif
// epilogue warps per CTA: 4 (one per TMEM lane quadrant) or 8 (two per
// quadrant, each on half of the item's columns: twice the C loads in flight)
constexpr int EPI_WARPS = MT_TC2_EPI;
constexpr int EPI_COLS = BN / (EPI_WARPS / 4);
constexpr int NUM_THREADS = 64 + 32 * EPI_WARPS;
constexpr int EPI_STRIDE = 33;
constexpr int CSLOTS = 4, CSLOT_BYTES = 32 * 32 * 4;  // TMA epilogue: per-warp C chunk ring
constexpr int EPI_BYTES = MT_TC2_TMAEPI ? EPI_WARPS * CSLOTS * CSLOT_BYTES
                                        : EPI_WARPS * 32 * EPI_STRIDE * 4;
static_assert(!MT_TC2_TMAEPI || EPI_WARPS == 4, "TMA epilogue assumes one warp per TMEM quadrant");
constexpr int TMEM_COLS = 512;        // 2 accumulators x 256 columns
constexpr int SCHED = 4;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 640;

// kind::tf32, D f32, A/B tf32 K-major, N = 256, M = 256 (cta_group::2)
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(256 >> 4) << 24);

}  // namespace
#include "tc2_common.cuh"
namespace {
using namespace mt_tma;
using namespace mt_pair;
// v[u] += (correction accumulator, 32 columns at taddr) in FP32 round-to-nearest
__device__ __forceinline__ void add_corr(uint32_t (&v)[32], uint32_t taddr) {
  uint32_t w[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
        "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]),
        "=r"(w[14]), "=r"(w[15]), "=r"(w[16]), "=r"(w[17]), "=r"(w[18]), "=r"(w[19]), "=r"(w[20]),
        "=r"(w[21]), "=r"(w[22]), "=r"(w[23]), "=r"(w[24]), "=r"(w[25]), "=r"(w[26]), "=r"(w[27]),
        "=r"(w[28]), "=r"(w[29]), "=r"(w[30]), "=r"(w[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int u = 0; u < 32; ++u) v[u] = __float_as_uint(__uint_as_float(v[u]) + __uint_as_float(w[u]));
}
__device__ __forceinline__ void umma2_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}

struct Work2 {
  int64_t slot0;
  int nitems;    // slots * nsubm * nsubn (pair items of 256 x 256)
  int nsubm, nsubn;
  int* counter;  // [work queue head, pairs started]
  int presplit;
  unsigned long long* span;  // profiling: device-side [start, end] stamps (or null)
  int mlo, mhi, sw;          // update: owned column range and super-column width (0 = slot order)
};

template <bool TRSM>
__device__ __forceinline__ void tc2_body(const Grid& g, int k, const Work2& w,
                                         const CUtensorMap& map_a, const CUtensorMap& map_b,
                                         const CUtensorMap& map_c) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  float* epi = (float*)(smem + STAGES * STAGE_BYTES);
  uint64_t* full = (uint64_t*)(smem + STAGES * STAGE_BYTES + EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;
  uint64_t* sempty = sfull + SCHED;
  int* sitem = (int*)(sempty + SCHED);
  int* si = sitem + SCHED;  // tile row i of the item
  int* sj = si + SCHED;     // tile column j of the item
  uint64_t* cbar = (uint64_t*)(sj + SCHED);  // TMA epilogue: C chunk slots, CSLOTS per warp
  uint32_t* tmem_slot = (uint32_t*)(cbar + EPI_WARPS * CSLOTS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // co-scheduled band update (option 10): once every pair of this grid is
  // resident, a programmatic-dependent DMMA launch may take the SMs left over
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const int nb = g.nb;
  const int nsub = w.nsubm * w.nsubn;
  auto item_ksteps = [&](int item) {
    return TRSM ? ((item % nsub) % w.nsubn + 1) * (BN / BK) : nb / BK;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);   // leader: its producer's arrive.expect_tx (both CTAs' bytes)
      mbar_init(&empty[s], 1);  // one multicast commit per use
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * EPI_WARPS);  // leader: local + peer epilogue warps
    }
    for (int s = 0; s < SCHED; ++s) {
      mbar_init(&sfull[s], 1);
      mbar_init(&sempty[s], 2 + 2 * EPI_WARPS);  // leader: MMA + epi + peer producer + peer epi
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
  cluster_sync();  // barriers of both CTAs initialised before any remote arrive
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (w.span && threadIdx.x == 0) atomicMin(&w.span[0], mt_globaltimer());
  const uint32_t tmem_base = *tmem_slot;

  auto tile_of = [&](int item, int& i, int& j) {
    if (!TRSM && w.sw > 0) super_tile_ij(g, item / nsub, w.mlo, w.mhi, w.sw, i, j);
    else g.off_slot_ij(w.slot0 + item / nsub, i, j);
  };
  // consumer side of the work ring (both CTAs); the peer releases the
  // leader's slot remotely
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
    // release the slot with a relaxed arrive (no fence on this warp's pending C
    // stores); the shuffle makes the arrive depend on every lane's loaded values
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
      if (leader && !TRSM && g.yield) atomicAdd(w.counter + 1, 1);  // pairs started
      const int npairs = (int)(gridDim.x / 2);
      uint32_t it = 0;
      for (uint32_t li = 0;; ++li) {
        const int s = li % SCHED;
        int item, i = 0, j = 0;
        if (leader) {
          mbar_wait(&sempty[s], ((li / SCHED) & 1) ^ 1);
          // the pair stops on a failed pivot or on an SM-yield request (only while
          // some pair has not started: that one will drain the queue)
          if (g.failed()) {
            item = -1;
          } else if (!TRSM && g.yield && *(volatile int*)g.yield > 0 &&
                     *(volatile int*)(w.counter + 1) < npairs && atomicSub(g.yield, 2) > 0) {
            item = -1;
          } else {
            item = atomicAdd(w.counter, 1);
            if (item >= w.nitems) item = -1;
          }
          if (item >= 0) tile_of(item, i, j);
          sitem[s] = item; si[s] = i; sj[s] = j;
          st_cl_u32(peer_addr(&sitem[s], 1), (uint32_t)item);
          st_cl_u32(peer_addr(&si[s], 1), (uint32_t)i);
          st_cl_u32(peer_addr(&sj[s], 1), (uint32_t)j);
          mbar_arrive(&sfull[s]);
          mbar_arrive_cl(peer_addr(&sfull[s], 1));  // release: the peer sees the item
        } else {
          mbar_wait_cl(&sfull[s], (li / SCHED) & 1);
          item = *(volatile int*)&sitem[s];
          i = *(volatile int*)&si[s];
          j = *(volatile int*)&sj[s];
          if ((item ^ i ^ j) != 0x7fffffff) mbar_arrive_cl_relaxed(peer_addr(&sempty[s], 0));
        }
        if (item < 0) break;
        const int sub = item % nsub;
        const int m0 = (sub / w.nsubn) * (2 * BM) + (int)rank * BM;
        const int n0 = (sub % w.nsubn) * BN + (int)rank * BNH;
        // split buffer rows: hi of tile (i, k) at ((k&1)*p + i)*2*nb, lo at + nb;
        // TRSM: A = pre-split of B_ik, B = split of W = L_kk^{-1}
        const int arow = TRSM ? (int)g.presplit_row(i) + m0 : (int)g.split_row(i, k) + m0;
        const int brow = TRSM ? (int)g.winv_row() + n0 : (int)g.split_row(j, k) + n0;
        const int ksteps = item_ksteps(item);
        for (int ks = 0; ks < ksteps; ++ks, ++it) {
          const int st = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty[st], ph ^ 1);
          unsigned char* sb = smem + st * STAGE_BYTES;
          if (leader) mbar_expect_tx(&full[st], 2 * STAGE_BYTES);
          const uint32_t bar = peer_addr(&full[st], 0);
          tma_load_pair(sb, &map_a, bar, ks * BK, arow);                               // A hi
          tma_load_pair(sb + A_BYTES, &map_b, bar, ks * BK, brow);                     // B hi
          tma_load_pair(sb + A_BYTES + B_BYTES, &map_a, bar, ks * BK, arow + nb);      // A lo
          tma_load_pair(sb + 2 * A_BYTES + B_BYTES, &map_b, bar, ks * BK, brow + nb);  // B lo
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
        const int ksteps = item_ksteps(item);
        const uint32_t b = li & 1, aph = (li >> 1) & 1;
        mbar_wait_cl(&tempty[b], aph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t dcol = tmem_base + b * ACC_STRIDE;
        const uint32_t ccol = MT_TC2_SPLITACC ? dcol + BN : dcol;  // correction accumulator
        for (int ks = 0; ks < ksteps; ++ks, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (lane == 0) {
            unsigned char* st = smem + s * STAGE_BYTES;
            const unsigned char* ahi = st;
            const unsigned char* bhi = st + A_BYTES;
            const unsigned char* alo = st + A_BYTES + B_BYTES;
            const unsigned char* blo = alo + A_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const int off = kk * 32;  // 8 fp32 along K = 32 B inside the 64 B swizzle row
              const uint32_t first = (ks == 0 && kk == 0) ? 0u : 1u;
              umma2_tf32(ccol, sw64_desc(alo + off), sw64_desc(bhi + off), first);
              umma2_tf32(ccol, sw64_desc(ahi + off), sw64_desc(blo + off), 1u);
              umma2_tf32(dcol, sw64_desc(ahi + off), sw64_desc(bhi + off),
                         MT_TC2_SPLITACC ? first : 1u);
            }
            umma2_commit_both(&empty[s]);                        // both CTAs' stage s free
            if (ks == ksteps - 1) umma2_commit_both(&tfull[b]);  // both accumulators ready
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2..5, both CTAs)
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int c_lo = EPI_WARPS == 4 ? 0 : ((warp - 2) / 4) * EPI_COLS;  // this warp's columns
    const uint32_t tempty_leader[2] = {peer_addr(&tempty[0], 0), peer_addr(&tempty[1], 0)};
#if MT_TC2_TMAEPI
    unsigned char* wslots = (unsigned char*)epi + (warp - 2) * CSLOTS * CSLOT_BYTES;
    uint64_t* wbar = cbar + (warp - 2) * CSLOTS;
    float* stg = (float*)wslots;  // register-path transpose buffer aliases the slots
    uint32_t gl = 0, gu = 0;      // C chunks loaded / used by this warp (slot = n % CSLOTS)
#else
    float* stg = epi + (warp - 2) * 32 * EPI_STRIDE;
#endif
    for (uint32_t li = 0;; ++li) {
      int i, j;
      const int item = next_item(li, &i, &j);
      if (item < 0) break;
      const int sub = item % nsub;
      const int m0 = (sub / w.nsubn) * (2 * BM) + (int)rank * BM, n0 = (sub % w.nsubn) * BN;
      const uint32_t b = li & 1, aph = (li >> 1) & 1;
      const int64_t roff = (int64_t)(m0 + q * 32) * nb + n0;
      float* cbase = g.stile(i, j) + roff;
#if MT_TC2_TMAEPI
      if (!TRSM && !(w.presplit && j == k + 1)) {
        // ---- TMA path: C chunk (32 rows x 32 columns, SWIZZLE_128B) per slot;
        // lane = row, matching the tcgen05.ld 32x32b layout (no transpose)
        const int crow = (int)((g.scol(j) + (i - j - g.t)) * (int64_t)nb) + m0 + q * 32;
        auto load_chunk = [&](int c, int newer) {  // newer: stores issued after the slot's last one
          if (lane == 0) {
            if (newer >= 3) bulk_wait_read<3>();
            else if (newer == 2) bulk_wait_read<2>();
            else if (newer == 1) bulk_wait_read<1>();
            else bulk_wait_read<0>();
            const uint32_t s = gl % CSLOTS;
            mbar_expect_tx(&wbar[s], CSLOT_BYTES);
            tma_load_2d(wslots + s * CSLOT_BYTES, &map_c, &wbar[s], n0 + c * 32, crow);
          }
          ++gl;
        };
        for (int c = 0; c < 3; ++c) load_chunk(c, (int)gu - (int)gl + 3);
        mbar_wait(&tfull[b], aph);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + b * ACC_STRIDE;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
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
              : "r"(taddr + c * 32));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (MT_TC2_SPLITACC) add_corr(v, taddr + BN + c * 32);
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
            tma_store_2d(&map_c, wslots + s * CSLOT_BYTES, n0 + c * 32, crow);
            bulk_commit();
          }
          ++gu;
          if (c + 3 < BN / 32) load_chunk(c + 3, (int)gu - (int)gl + 3);
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive_cl_relaxed(tempty_leader[b]);
        continue;
      }
      // register path (TRSM, or the column-(k+1) update with its split outputs):
      // its transpose buffer aliases the chunk slots -> drain the TMA stores first
      if (lane == 0) bulk_wait_all();
      __syncwarp();
#endif
      float cn[32];
      if constexpr (!TRSM) {
#pragma unroll
        for (int r = 0; r < 32; ++r) cn[r] = cbase[(int64_t)r * nb + c_lo + lane];
      }
      mbar_wait(&tfull[b], aph);
      asm volatile("tcgen05.fence::after_thread_sync;");
      float* shi = TRSM ? g.split_hi(i, k) + roff
                        : ((w.presplit && j == k + 1) ? g.presplit_hi(i) + roff : nullptr);
      const int64_t te = g.tile_elems();
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + b * ACC_STRIDE;
#pragma unroll 1
      for (int c = c_lo; c < c_lo + EPI_COLS; c += 32) {
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
            : "r"(taddr + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (MT_TC2_SPLITACC) add_corr(v, taddr + BN + c);
#pragma unroll
        for (int u = 0; u < 32; ++u) stg[lane * EPI_STRIDE + u] = __uint_as_float(v[u]);
        __syncwarp();
        float* cp = cbase + c + lane;
        float cv[32];
        if constexpr (TRSM) {
#pragma unroll
          for (int r = 0; r < 32; ++r) cv[r] = stg[r * EPI_STRIDE + lane];
        } else {
#pragma unroll
          for (int r = 0; r < 32; ++r) cv[r] = cn[r];
          if (c + 32 < c_lo + EPI_COLS) {
#pragma unroll
            for (int r = 0; r < 32; ++r) cn[r] = cp[(int64_t)r * nb + 32];
          }
#pragma unroll
          for (int r = 0; r < 32; ++r) cv[r] -= stg[r * EPI_STRIDE + lane];
        }
#pragma unroll
        for (int r = 0; r < 32; ++r) cp[(int64_t)r * nb] = cv[r];
        if (shi) {
          float* hrow = shi + c + lane;
#pragma unroll
          for (int r = 0; r < 32; ++r) {
            float h, l;
            mt_tf32_split(cv[r], h, l);
            asm volatile("st.global.f32 [%0], %1;" ::"l"(hrow), "f"(h) : "memory");
            asm volatile("st.global.f32 [%0], %1;" ::"l"(hrow + te), "f"(l) : "memory");
            asm volatile("" : "+l"(hrow));
            hrow += nb;
          }
        }
        __syncwarp();
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      // TMEM reads completed (tcgen05.wait::ld): relaxed arrive, no wait on the C stores
      if (lane == 0) mbar_arrive_cl_relaxed(tempty_leader[b]);
#if MT_TC2_TMAEPI
      // the transpose buffer's generic writes precede later TMA refills of the slots
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
    }
#if MT_TC2_TMAEPI
    if (lane == 0) bulk_wait_all();  // C stores complete before the kernel ends
    __syncwarp();
#endif
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();  // no remote arrive / MMA of the pair still targets this CTA
  if (w.span && threadIdx.x == 0) atomicMax(&w.span[1], mt_globaltimer());
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    tc2_update_kernel(Grid g, int k, Work2 w, const __grid_constant__ CUtensorMap map_a,
                      const __grid_constant__ CUtensorMap map_b,
                      const __grid_constant__ CUtensorMap map_c) {
  tc2_body<false>(g, k, w, map_a, map_b, map_c);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    tc2_trsm_kernel(Grid g, int k, Work2 w, const __grid_constant__ CUtensorMap map_a,
                    const __grid_constant__ CUtensorMap map_b,
                    const __grid_constant__ CUtensorMap map_c) {
  tc2_body<true>(g, k, w, map_a, map_b, map_c);
}

int g_sm2 = 0;

}  // namespace

// launch over the off-band slot range [s0, s0 + scnt) of step k; `ctas` caps
// the grid (rounded down to pairs)
int mt_tc2_launch(const Grid& g, int k, int64_t s0, int64_t scnt, int ctas, bool trsm,
                  int presplit, cudaStream_t st, unsigned long long* span, int jlo, int jhi) {
  if (scnt <= 0) return MT_OK;
  CUtensorMap ma, mb;
  const int64_t split_rows = g.split_rows();
  int rc = make_map_2d(&ma, g.split, split_rows, g.nb, 4, BK, BM, CU_TENSOR_MAP_SWIZZLE_64B);
  if (!rc) rc = make_map_2d(&mb, g.split, split_rows, g.nb, 4, BK, BNH, CU_TENSOR_MAP_SWIZZLE_64B);
  // C (off-band pool) in 32 x 32 FP32 chunks for the TMA epilogue
  CUtensorMap mc;
  const int64_t c_rows = g.noff() > 0 ? g.noff() * g.nb : 32;
  if (!rc) rc = make_map_2d(&mc, g.sp ? (const void*)g.sp : (const void*)g.split, c_rows, g.nb, 4, 32,
                            32, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  Work2 w;
  w.slot0 = s0;
  w.nsubm = g.nb / (2 * BM);
  w.nsubn = g.nb / BN;
  w.nitems = (int)(scnt * w.nsubm * w.nsubn);
  w.presplit = presplit;
  w.span = span;
  w.mlo = g.owned_before(jlo);
  w.mhi = g.owned_before(jhi);
  w.sw = (!trsm && jhi > jlo + 1 && g.rs == 1) ? mt_opt_super_cols() : 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!g_sm2) cudaDeviceGetAttribute(&g_sm2, cudaDevAttrMultiProcessorCount, dev);
  static int* counters[64] = {nullptr};
  static unsigned next_counter[64] = {0};
  if (dev < 0 || dev >= 64) { mt_set_error("device index out of range"); return MT_E_CUDA; }
  if (!counters[dev] && mt_cuda_check(cudaMalloc(&counters[dev], 2 * 256 * sizeof(int)), "counter alloc"))
    return MT_E_CUDA;
  w.counter = counters[dev] + 2 * (next_counter[dev]++ % 256);
  if (mt_cuda_check(cudaMemsetAsync(w.counter, 0, 2 * sizeof(int), st), "counter reset"))
    return MT_E_CUDA;
  int pairs = (ctas > 0 ? ctas : g_sm2) / 2;
  if (!trsm && g.yield && ctas <= 0) pairs = g_sm2;  // oversubscribed: refills yielded SMs
  if (pairs > w.nitems) pairs = w.nitems;
  if (pairs < 1) pairs = 1;
  const size_t smem = SMEM_BYTES;
  if (trsm) {
    cudaFuncSetAttribute(tc2_trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    tc2_trsm_kernel<<<2 * pairs, NUM_THREADS, smem, st>>>(g, k, w, ma, mb, mc);
    MT_LAUNCH_CHECK("tc2_trsm_kernel");
  } else {
    cudaFuncSetAttribute(tc2_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    tc2_update_kernel<<<2 * pairs, NUM_THREADS, smem, st>>>(g, k, w, ma, mb, mc);
    MT_LAUNCH_CHECK("tc2_update_kernel");
  }
  return MT_OK;
}
