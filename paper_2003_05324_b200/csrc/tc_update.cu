// FP32 (off-band) trailing update on the 5th-gen tensor cores: 3xTF32.
//
//   C_ij <- C_ij - A_ik A_jk^T      (kernels.gemm FP32 path, factor.py:273-274)
//
// FP32 products are emulated with three TF32 UMMAs per K-step,
//   A B^T ~= A_lo B_hi^T + A_hi B_lo^T + A_hi B_hi^T,
// hi = cvt.rna.tf32(x) (exactly representable in TF32), lo = x - hi (exact
// in FP32; Grid-level helper mt_tf32_split).  The dropped A_lo B_lo term and
// the TF32 truncation of lo are O(2^-22) relative, i.e. FP32-class accuracy:
// measured factor error vs the CPU reference 0.4-0.95x that of the SIMT FFMA
// kernel (tools/acc_tf32.py; bounded in tests/test_gpu_tc.py).  The hi/lo split is
// produced once per panel tile by the TRSM epilogue (Grid::split_hi/lo), so
// the update streams both halves straight from L2 with TMA -- no per-stage
// conversion through the LSU pipe.
//
// Structure (one CTA per SM, persistent over the step's 128x256 work items):
//   warp 0      TMA producer: 16-wide K slabs of A_hi, B_hi, A_lo, B_lo
//               (SWIZZLE_64B), 4-stage mbarrier ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128,
//               N=256, K=8, kind::tf32), commits to mbarriers
//   warps 2-5   epilogue: tcgen05.ld 32 columns/thread, transposed through
//               shared memory, coalesced C -= acc in HBM; TMEM is
//               double-buffered so it overlaps the next item's MMAs
// Work items are ordered by output tile, so concurrently running CTAs share
// panel tiles in L2.  Every output element is written by one CTA per step in
// ascending k: deterministic, schedule-invariant.
#include <cuda.h>

#include "tma.cuh"

namespace {
using namespace mt_tma;

constexpr int BM = 128, BN = 256, BK = 16, STAGES = 4;
constexpr int A_BYTES = BM * BK * 4;          // 8 KB
constexpr int B_BYTES = BN * BK * 4;          // 16 KB
constexpr int STAGE_BYTES = 2 * (A_BYTES + B_BYTES);  // hi + lo = 48 KB
#ifndef MT_EPI_WARPS
#define MT_EPI_WARPS 4
#endif
// epilogue warps: 4 (one per TMEM lane quadrant) or 8 (two per quadrant, each
// taking half of the item's columns: twice the C loads in flight)
constexpr int EPI_WARPS = MT_EPI_WARPS;
constexpr int EPI_COLS = BN / (EPI_WARPS / 4);
constexpr int NUM_THREADS = 64 + 32 * EPI_WARPS;
constexpr int EPI_STRIDE = 33;                                // transpose tile, conflict-free
constexpr int EPI_BYTES = EPI_WARPS * 32 * EPI_STRIDE * 4;    // per warp 32x33 floats
constexpr int TMEM_COLS = 512;                // 2 accumulators x 256 columns

// K-major, SWIZZLE_64B smem matrix descriptor (8-row atoms of 64 B, SBO = 512 B)
__device__ __forceinline__ uint64_t sw64_desc(const void* p) {
  const uint64_t a = (smem_u32(p) >> 4) & 0x3FFF;
  return a | ((uint64_t)(512 >> 4) << 32) | (1ull << 46) | (4ull << 61);
}
// kind::tf32, D f32, A/B tf32 K-major, N = 256, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

struct Work {
  int64_t slot0;
  int nitems;  // slots * nsub
  int nsubm, nsubn;
  int* counter;  // [dynamic work queue head, CTAs started] (zeroed before the launch)
  int presplit;  // update: also write the pre-TRSM split of column k+1 outputs
  int mlo, mhi;  // update: owned tile-column index range [mlo, mhi) of the outputs
  int sw;        // update: super-column width (owned columns); 0 = slot order
  int l2pf;      // update: prefetch each item's C block into L2 when it is dequeued
  int diag;      // diagnostics only (option 8): 1 skip C loads, 2 skip C stores, 4 skip epilogue
};

constexpr int SCHED = 4;  // work-item ring between the producer and the consumers

// TRSM = false: C_ij -= A_ik A_jk^T (trailing update of step k)
// TRSM = true:  X_ik = B_ik W^T, W = L_kk^{-1} (off-band panel solve of step k):
//               A rows from the pre-split of B, B rows from the split of W; W is
//               lower triangular, so output columns [n0, n0 + 256) need K < n0 + 256
template <bool TRSM>
__device__ __forceinline__ void tc32_body(const Grid& g, int k, const Work& w,
                                          const CUtensorMap& map_a, const CUtensorMap& map_b) {
  if (g.failed()) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem =
      (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);  // SW64 needs 512B+
  float* epi = (float*)(smem + STAGES * STAGE_BYTES);
  uint64_t* full = (uint64_t*)(smem + STAGES * STAGE_BYTES + EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;
  uint64_t* sempty = sfull + SCHED;
  int* sitem = (int*)(sempty + SCHED);
  int2* sij = (int2*)(sitem + SCHED);  // (i, j) of the item, computed once by the producer
  uint32_t* tmem_slot = (uint32_t*)(sij + SCHED);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = g.nb;
  const int nsub = w.nsubm * w.nsubn;
  auto item_ksteps = [&](int item) {
    return TRSM ? ((item % nsub) % w.nsubn + 1) * (BN / BK) : nb / BK;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], EPI_WARPS);
    }
    for (int s = 0; s < SCHED; ++s) {
      mbar_init(&sfull[s], 1);
      mbar_init(&sempty[s], 1 + EPI_WARPS);  // MMA warp + epilogue warps release a slot
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_base = *tmem_slot;

  auto item_ij = [&](int item, int& i, int& j, int& m0, int& n0) {
    const int64_t tile = item / nsub;
    const int sub = item % nsub;
    if (!TRSM && w.sw > 0) super_tile_ij(g, tile, w.mlo, w.mhi, w.sw, i, j);
    else g.off_slot_ij(w.slot0 + tile, i, j);
    m0 = (sub / w.nsubn) * BM;
    n0 = (sub % w.nsubn) * BN;
  };
  // consumers read the li-th work item (and its tile) from the ring (-1 = no more work)
  auto next_item = [&](uint32_t li, int2* ij) {
    const int s = li % SCHED;
    mbar_wait(&sfull[s], (li / SCHED) & 1);
    const int item = *(volatile int*)&sitem[s];
    int dep = item;
    if (ij) {
      ij->x = *(volatile int*)&sij[s].x;
      ij->y = *(volatile int*)&sij[s].y;
      dep ^= ij->x ^ ij->y;
    }
    // relaxed release of the slot, dependent on every lane's loaded values
    dep = __reduce_xor_sync(0xffffffffu, dep);
    if ((threadIdx.x & 31) == 0 && dep != 0x7fffffff) mbar_arrive_relaxed(&sempty[s]);
    return item;
  };

  if (warp == 0) {
    // ------------------------------------------------ TMA producer + work queue
    if (lane == 0) {
      if (!TRSM && g.yield) atomicAdd(w.counter + 1, 1);  // CTAs started
      uint32_t it = 0;
      for (uint32_t li = 0;; ++li) {
        const int s = li % SCHED;
        mbar_wait(&sempty[s], ((li / SCHED) & 1) ^ 1);
        // SM-yield request from the panel stream: this CTA stops taking work
        // (an oversubscribed grid refills the SM once the panel kernels ran)
        // A CTA may only yield while some CTA of the grid has not started yet:
        // that one is guaranteed to run later and drain the queue.
        int item;
        if (!TRSM && g.yield && *(volatile int*)g.yield > 0 &&
            *(volatile int*)(w.counter + 1) < (int)gridDim.x && atomicSub(g.yield, 1) > 0) {
          item = -1;
        } else {
          item = atomicAdd(w.counter, 1);
          if (item >= w.nitems) item = -1;
        }
        int i = 0, j = 0, m0 = 0, n0 = 0;
        if (item >= 0) item_ij(item, i, j, m0, n0);
        sitem[s] = item;
        sij[s] = make_int2(i, j);
        mbar_arrive(&sfull[s]);  // release: consumers see sitem[s], sij[s]
        if (item < 0) break;
        if (!TRSM && w.l2pf) {
          // stage this item's C block (128 rows x 1 KB) in L2: the epilogue reads
          // it one item later, so its loads hit L2 instead of waiting on HBM
          const float* crow = g.stile(i, j) + (int64_t)m0 * nb + n0;
          for (int r = 0; r < BM; ++r, crow += nb)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(crow), "r"(BN * 4)
                         : "memory");
        }
        // split buffer rows: hi of tile (i, k) at ((k&1)*p + i)*2*nb, lo at + nb;
        // TRSM: A = pre-split of B_ik, B = split of W = L_kk^{-1}
        const int arow = TRSM ? (int)g.presplit_row(i) + m0 : (int)g.split_row(i, k) + m0;
        const int brow = TRSM ? (int)g.winv_row() + n0 : (int)g.split_row(j, k) + n0;
        const int ksteps = item_ksteps(item);
        for (int ks = 0; ks < ksteps; ++ks, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          unsigned char* st = smem + s * STAGE_BYTES;
          mbar_expect_tx(&full[s], STAGE_BYTES);
          tma_load_2d(st, &map_a, &full[s], ks * BK, arow);                       // A hi
          tma_load_2d(st + A_BYTES, &map_b, &full[s], ks * BK, brow);             // B hi
          tma_load_2d(st + A_BYTES + B_BYTES, &map_a, &full[s], ks * BK, arow + nb);   // A lo
          tma_load_2d(st + 2 * A_BYTES + B_BYTES, &map_b, &full[s], ks * BK, brow + nb);  // B lo
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    uint32_t it = 0;
    for (uint32_t li = 0;; ++li) {
      const int item = next_item(li, nullptr);
      if (item < 0) break;
      const int ksteps = item_ksteps(item);
      const uint32_t b = li & 1, aph = (li >> 1) & 1;
      mbar_wait(&tempty[b], aph ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t dcol = tmem_base + b * BN;
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
            umma_tf32(dcol, sw64_desc(alo + off), sw64_desc(bhi + off), first);
            umma_tf32(dcol, sw64_desc(ahi + off), sw64_desc(blo + off), 1u);
            umma_tf32(dcol, sw64_desc(ahi + off), sw64_desc(bhi + off), 1u);
          }
          umma_commit(&empty[s]);                          // stage free when these finish
          if (ks == ksteps - 1) umma_commit(&tfull[b]);    // accumulator ready
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2..5)
    // C is read from HBM one 32x32 chunk ahead of its use, the first chunk
    // before the accumulator wait, so the load latency overlaps the MMAs
    // instead of pacing them.
    const int q = warp & 3;          // TMEM lane quadrant this warp may access
    float* stg = epi + (warp - 2) * 32 * EPI_STRIDE;
    const int c_lo = EPI_WARPS == 4 ? 0 : ((warp - 2) / 4) * EPI_COLS;  // column range of this warp
    for (uint32_t li = 0;; ++li) {
      int2 ij;
      const int item = next_item(li, &ij);
      if (item < 0) break;
      const int i = ij.x, j = ij.y;
      const int sub = item % nsub;
      const int m0 = (sub / w.nsubn) * BM, n0 = (sub % w.nsubn) * BN;
      const uint32_t b = li & 1, aph = (li >> 1) & 1;
      // rows q*32 .. q*32+31 of the 128x256 item; lane owns row q*32+lane in TMEM
      const int64_t roff = (int64_t)(m0 + q * 32) * nb + n0;
      float* cbase = g.stile(i, j) + roff;
      float cn[32];
      const int diag = w.diag;
      if constexpr (!TRSM) {
        if (!(diag & 1)) {
#pragma unroll
          for (int r = 0; r < 32; ++r) cn[r] = cbase[(int64_t)r * nb + c_lo + lane];
        } else {
#pragma unroll
          for (int r = 0; r < 32; ++r) cn[r] = 0.0f;
        }
      }
      mbar_wait(&tfull[b], aph);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (diag & 4) {
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
        continue;
      }
      // split outputs: TRSM -> the panel split read by this step's updates;
      // update of column k+1 -> the pre-TRSM split of the next panel
      float* shi = TRSM ? g.split_hi(i, k) + roff
                        : ((w.presplit && j == k + 1) ? g.presplit_hi(i) + roff : nullptr);
      const int64_t te = g.tile_elems();
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + b * BN;
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
        // transpose the 32x32 block through shared memory (row = lane -> column = lane)
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
          if (c + 32 < c_lo + EPI_COLS && !(diag & 1)) {
#pragma unroll
            for (int r = 0; r < 32; ++r) cn[r] = cp[(int64_t)r * nb + 32];
          }
#pragma unroll
          for (int r = 0; r < 32; ++r) cv[r] -= stg[r * EPI_STRIDE + lane];
        }
        if (!(diag & 2)) {
#pragma unroll
          for (int r = 0; r < 32; ++r) cp[(int64_t)r * nb] = cv[r];
        } else if (cv[0] == 1.2345f) {
          cp[0] = cv[31];  // keep the arithmetic live
        }
        if (shi) {
          float* hrow = shi + c + lane;
#pragma unroll
          for (int r = 0; r < 32; ++r) {
            float h, l;
            mt_tf32_split(cv[r], h, l);
            asm volatile("st.global.f32 [%0], %1;" ::"l"(hrow), "f"(h) : "memory");
            asm volatile("st.global.f32 [%0], %1;" ::"l"(hrow + te), "f"(l) : "memory");
            asm volatile("" : "+l"(hrow));  // keep one running row pointer (no hoisted addresses)
            hrow += nb;
          }
        }
        __syncwarp();
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive_relaxed(&tempty[b]);  // TMEM reads done; C stores need no fence
    }
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
    tc32_update_kernel(Grid g, int k, Work w, const __grid_constant__ CUtensorMap map_a,
                       const __grid_constant__ CUtensorMap map_b) {
  tc32_body<false>(g, k, w, map_a, map_b);
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
    tc32_trsm_kernel(Grid g, int k, Work w, const __grid_constant__ CUtensorMap map_a,
                     const __grid_constant__ CUtensorMap map_b) {
  tc32_body<true>(g, k, w, map_a, map_b);
}

// ------------------------------------------------------------- host side
int make_map(CUtensorMap* m, const float* base, int64_t rows, int nb, int box_rows) {
  return make_map_2d(m, base, rows, nb, 4, BK, box_rows, CU_TENSOR_MAP_SWIZZLE_64B);
}

int g_sm_count = 0;

}  // namespace

namespace mt_tma {
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

int make_map_2d(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int es,
                int box_cols, int box_rows, CUtensorMapSwizzle swz) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) { mt_set_error("cuTensorMapEncodeTiled unavailable"); return MT_E_CUDA; }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)(rows > 0 ? rows : 1)};
  cuuint64_t strides[1] = {(cuuint64_t)cols * es};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, es == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                  2, (void*)base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    mt_set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return MT_E_CUDA;
  }
  return MT_OK;
}
}  // namespace mt_tma

bool mt_tc_supported(const Grid& g) {
  return g.mode == MT_MODE_MP && g.split != nullptr && g.nb % BN == 0 &&
         g.split_rows() < (1ll << 31);
}

bool mt_tc_trsm_enabled(const Grid& g) {
  return mt_opt_tc_trsm() && (mt_engine_tc(mt_opt_engine()) || g.multi()) &&
         mt_tc_supported(g);
}

namespace {
// persistent launch over `nitems` work items of slot range [s0, s0 + scnt)
int launch_tc32(const Grid& g, int k, int64_t s0, int64_t scnt, int ctas, bool trsm,
                cudaStream_t st, int jlo = 0, int jhi = 0, unsigned long long* span = nullptr) {
  if (scnt <= 0) return MT_OK;
  // default engine: round-to-nearest chunked accumulation (tcf_update.cu); the
  // kernels below accumulate the whole K range in TMEM (opt-in engine 2)
  if (mt_opt_engine() != MT_ENGINE_TF32X3_RZ)
    return mt_tcf_launch(g, k, s0, scnt, ctas, trsm, (!trsm && mt_tc_trsm_enabled(g)) ? 1 : 0, st,
                         span, jlo, jhi);
  // full-width (256 x 512) CTA-pair items for the bulk update (tc2w_update.cu)
  if (!trsm && mt_opt_wide_items() && mt_opt_cta_pairs() && mt_tc2w_supported(g) && jlo > k + 1 &&
      !mt_opt_tc_diag() && !mt_opt_c_prefetch())
    return mt_tc2w_launch(g, k, s0, scnt, ctas, st, span);
  if (mt_opt_cta_pairs() && !mt_opt_tc_diag() && !mt_opt_c_prefetch())  // CTA-pair kernel
    return mt_tc2_launch(g, k, s0, scnt, ctas, trsm,
                         (!trsm && mt_tc_trsm_enabled(g)) ? 1 : 0, st, span, jlo, jhi);
  CUtensorMap ma, mb;
  const int64_t split_rows = g.split_rows();  // whole split buffer
  int rc = make_map(&ma, g.split, split_rows, g.nb, BM);
  if (!rc) rc = make_map(&mb, g.split, split_rows, g.nb, BN);
  if (rc) return rc;
  Work w;
  w.slot0 = s0;
  w.nsubm = g.nb / BM;
  w.nsubn = g.nb / BN;
  w.nitems = (int)(scnt * w.nsubm * w.nsubn);
  w.presplit = (!trsm && mt_tc_trsm_enabled(g)) ? 1 : 0;
  w.mlo = g.owned_before(jlo);
  w.mhi = g.owned_before(jhi);
  w.sw = (!trsm && jhi > jlo && g.rs == 1) ? mt_opt_super_cols() : 0;
  w.l2pf = trsm ? 0 : mt_opt_c_prefetch();
  w.diag = trsm ? 0 : mt_opt_tc_diag();
  int dev = 0;
  cudaGetDevice(&dev);
  if (!g_sm_count) cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
  // per-launch work-queue head: a rotating slot of a small per-device buffer
  static int* counters[64] = {nullptr};
  static unsigned next_counter[64] = {0};
  if (dev < 0 || dev >= 64) { mt_set_error("device index out of range"); return MT_E_CUDA; }
  // per launch: [queue head, CTAs started]
  if (!counters[dev] && mt_cuda_check(cudaMalloc(&counters[dev], 2 * 256 * sizeof(int)), "counter alloc"))
    return MT_E_CUDA;
  w.counter = counters[dev] + 2 * (next_counter[dev]++ % 256);
  if (mt_cuda_check(cudaMemsetAsync(w.counter, 0, 2 * sizeof(int), st), "counter reset"))
    return MT_E_CUDA;
  int grid = ctas > 0 ? ctas : g_sm_count;
  if (!trsm && g.yield && ctas <= 0) grid = 2 * g_sm_count;  // room to refill yielded SMs
  if (grid > w.nitems) grid = w.nitems;
  const size_t smem = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 256 + SCHED * 8;
  if (trsm) {
    cudaFuncSetAttribute(tc32_trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    tc32_trsm_kernel<<<grid, NUM_THREADS, smem, st>>>(g, k, w, ma, mb);
    MT_LAUNCH_CHECK("tc32_trsm_kernel");
  } else {
    cudaFuncSetAttribute(tc32_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    tc32_update_kernel<<<grid, NUM_THREADS, smem, st>>>(g, k, w, ma, mb);
    MT_LAUNCH_CHECK("tc32_update_kernel");
  }
  return MT_OK;
}
}  // namespace

// FP32 updates of step k into off-band slots [s0, s0+scnt) via tcgen05; `ctas` caps the grid.
int mt_tc_update_impl(const Grid& g, int k, int jlo, int jhi, int ctas, cudaStream_t st,
                      unsigned long long* span) {
  const int64_t s0 = g.scol(jlo), scnt = g.scol(jhi) - s0;
  return launch_tc32(g, k, s0, scnt, ctas, false, st, jlo, jhi, span);
}

// Off-band panel TRSM of step k: X_ik = B_ik W^T for the off-band rows of
// column k, W = L_kk^{-1} split by trinv_kernel, B_ik pre-split by the update
// epilogue of step k-1 (or presplit_kernel); writes X and its split.
int mt_tc_trsm_impl(const Grid& g, int k, cudaStream_t st) {
  const int64_t s0 = g.scol(k), cnt = g.scol(k + 1) - s0;
  if (cnt <= 0) return MT_OK;
  // algorithmic work as the reference's strsm: rows(i) * rows(k)^2 per tile
  const double nb = g.nb, rk = g.rows(k);
  const double rows_sum = (cnt - 1) * nb + g.rows(g.p - 1);
  ProfScope ps(MT_K_TRSM32, st, rows_sum * rk * rk, cnt * nb * nb * 4.0 * 5.0);
  return launch_tc32(g, k, s0, cnt, 0, true, st);
}
