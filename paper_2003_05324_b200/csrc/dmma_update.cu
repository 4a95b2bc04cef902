// FP64 band trailing update on the FP64 tensor-core pipe (SASS DMMA), with the
// operand K-slabs staged by TMA into shared memory through an mbarrier ring.
//
//   C_ij <- C_ij - A_ik A_jk^T   for band outputs i - j < t
//   (kernels.syrk / kernels.gemm FP64 paths, factor.py:266-272)
//
// Operands of panel k come in three storage kinds, fixed per CTA:
//   F64    FP64 band payload (dp pool; multi-GPU: the received panel ring)
//   F32    FP32 off-band payload (sp pool), widened exactly on the fragment load
//          (bit-identical to the reference's materialised widened copy,
//          factor.py:265, test_factor.py:146-153)
//   SPLIT  multi-GPU received off-band operand: TF32 hi/lo pair whose FP64 sum
//          is exactly the FP32 payload
// TMA boxes are 16 K-columns x 64 rows: FP64 rows are 128 B (SWIZZLE_128B),
// FP32 rows 64 B (SWIZZLE_64B); the fragment loads apply the same XOR so the
// m8n8k4 fragment reads are bank-conflict free.
//
// CTA tile 128 x 64, 8 warps of 32 x 32 (4 x 4 DMMA m8n8k4 fragments each),
// 4-stage ring of 16-wide K slabs, 2 CTAs per SM (epilogue of one CTA
// overlaps the other's MMAs).  Thread 0 is the producer: it refills a stage
// as soon as all 8 warps released it (one slab after they consumed it).  Every output element receives its K
// products in the same order (16-wide slabs, 4-wide DMMA steps) as the
// previous register-staged kernel: results are deterministic and identical
// on 1 or N GPUs.
#include "tma.cuh"

namespace {
using namespace mt_tma;

constexpr int BM = 128, BN = 64, BK = 16, ST = 4;
constexpr int A_REGION = BM * BK * 8;  // 16 KB (FP64 slab, or FP32 hi + lo)
constexpr int B_REGION = BN * BK * 8;  // 8 KB
constexpr int STAGE = A_REGION + B_REGION;
constexpr int SMEM = ST * STAGE + 1024 + 128;

enum Kind { KF64 = 0, KF32 = 1, KSPLIT = 2 };

struct Maps {
  CUtensorMap dp, sp, split, dpanel;  // box 16 x 64
};

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}

// element (r, kk) of a K-slab region (rows of 16 elements, shared-window
// address `base`) as FP64.  Explicit ld.shared: the stage is released with an
// mbarrier arrive right after these loads, and only shared-pipe loads are
// ordered before it (generic loads of the same data raced with the refill).
template <int KIND>
__device__ __forceinline__ double frag(uint32_t base, int r, int kk, int lo_off) {
  if constexpr (KIND == KF64) {
    const uint32_t off = r * 128 + ((((kk >> 1) ^ (r & 7)) << 4) | ((kk & 1) << 3));
    return lds_f64(base + off);
  } else {
    const uint32_t off = r * 64 + ((((kk >> 2) ^ ((r >> 1) & 3)) << 4) | ((kk & 3) << 2));
    double v = (double)lds_f32(base + off);
    if constexpr (KIND == KSPLIT) v += (double)lds_f32(base + lo_off + off);
    return v;
  }
}

struct Src {
  const CUtensorMap* map;
  int row;   // first row of the operand sub-block in the map's row space
  int lo;    // SPLIT: row offset of the lo half (nb)
  int kind;
};

__device__ __forceinline__ Src operand(const Grid& g, const Maps& maps, int i, int k, int r0) {
  Src s;
  s.lo = 0;
  if (g.band(i, k)) {
    s.kind = KF64;
    if (!g.multi()) {
      s.map = &maps.dp;
      s.row = (int)(g.dslot(i, k) * g.nb) + r0;
    } else {
      s.map = &maps.dpanel;
      s.row = (int)g.dpanel_row(i, k) + r0;
    }
  } else if (!g.multi()) {
    s.kind = KF32;
    s.map = &maps.sp;
    s.row = (int)(g.sslot(i, k) * g.nb) + r0;
  } else {
    s.kind = KSPLIT;
    s.map = &maps.split;
    s.row = (int)g.split_row(i, k) + r0;
    s.lo = g.nb;
  }
  return s;
}

__device__ __forceinline__ uint32_t region_bytes(int kind, int rows) {
  return kind == KF64 ? rows * BK * 8 : (kind == KF32 ? rows * BK * 4 : rows * BK * 8);
}

// issue the TMA loads of K slab ks for one operand (rows in boxes of 64)
__device__ __forceinline__ void load_operand(const Src& s, unsigned char* dst, int rows, int ks,
                                             uint64_t* bar) {
  const int rb = s.kind == KF64 ? 128 : 64;  // smem bytes per row
  for (int h = 0; h < rows; h += 64) {
    tma_load_2d(dst + h * rb, s.map, bar, ks * BK, s.row + h);
    if (s.kind == KSPLIT)
      tma_load_2d(dst + rows * 64 + h * rb, s.map, bar, ks * BK, s.row + s.lo + h);
  }
}

template <int KA, int KB>
__device__ __forceinline__ void mainloop(const unsigned char* smem, uint64_t* full, uint64_t* empty,
                                         const Src& a, const Src& b, int ksteps,
                                         double (&acc)[4][4][2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;
  const int fr = lane >> 2, fk = lane & 3;
  const int a_lo = BM * 64, b_lo = BN * 64;  // SPLIT: lo half after the hi half
  for (int ks = 0; ks < ksteps; ++ks) {
    const int s = ks % ST;
    mbar_wait(&full[s], (ks / ST) & 1);
    // Release the PREVIOUS stage only now: every DMMA of slab ks-1 was issued
    // before this wait loop, so their ld.shared operands have landed.  (An
    // arrive right after the loads may overtake them -- the scheduler hoists
    // it above the DMMAs -- and the refill TMA then races the reads.)
    if (ks > 0) {
      const int sp = (ks - 1) % ST;
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[sp]);
      // producer: refill it with slab ks - 1 + ST once every warp released it
      if (threadIdx.x == 0 && ks - 1 + ST < ksteps) {
        mbar_wait(&empty[sp], ((ks - 1) / ST) & 1);
        unsigned char* st = (unsigned char*)smem + sp * STAGE;
        mbar_expect_tx(&full[sp], region_bytes(a.kind, BM) + region_bytes(b.kind, BN));
        load_operand(a, st, BM, ks - 1 + ST, &full[sp]);
        load_operand(b, st + A_REGION, BN, ks - 1 + ST, &full[sp]);
      }
    }
    const uint32_t as = smem_u32(smem + s * STAGE);
    const uint32_t bs = as + A_REGION;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        af[f] = frag<KA>(as, wm + f * 8 + fr, k4 + fk, a_lo);
        bf[f] = frag<KB>(bs, wn + f * 8 + fr, k4 + fk, b_lo);
      }
#pragma unroll
      for (int fm = 0; fm < 4; ++fm)
#pragma unroll
        for (int fn = 0; fn < 4; ++fn) dmma884(acc[fm][fn], af[fm], bf[fn]);
    }
  }
}

__global__ void __launch_bounds__(256, 2)
    dmma_tma_update_kernel(Grid g, int k, int64_t slot0, int nsubm, int nsubn,
                           const __grid_constant__ Maps maps, unsigned long long* span) {
  if (span && threadIdx.x == 0) atomicMin(&span[0], mt_globaltimer());
  if (g.failed()) return;
  const int nsub = nsubm * nsubn;
  const int64_t slot = slot0 + blockIdx.x / nsub;
  const int sub = blockIdx.x % nsub;
  int i, j;
  g.band_slot_ij(slot, i, j);
  if (!g.present(i, k)) return;  // DST: GEMM(k; i, j) needs tile (i, k)
  const int m0 = (sub / nsubn) * BM, n0 = (sub % nsubn) * BN;
  const bool syrk = (i == j);
  if (syrk && n0 >= m0 + BM) return;  // entirely above the diagonal
  const int nb = g.nb, ksteps = nb / BK;

  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + ST * STAGE);
  uint64_t* empty = full + ST;

  const Src a = operand(g, maps, i, k, m0), b = operand(g, maps, j, k, n0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t tx = region_bytes(a.kind, BM) + region_bytes(b.kind, BN);
    for (int s = 0; s < ST && s < ksteps; ++s) {
      mbar_expect_tx(&full[s], tx);
      load_operand(a, smem + s * STAGE, BM, s, &full[s]);
      load_operand(b, smem + s * STAGE + A_REGION, BN, s, &full[s]);
    }
  }
  __syncthreads();

  double acc[4][4][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;

  // (A, B) kinds: band outputs have B band => A band, so B off-band implies A off-band
  if (a.kind == KF64 && b.kind == KF64) mainloop<KF64, KF64>(smem, full, empty, a, b, ksteps, acc);
  else if (a.kind == KF32 && b.kind == KF64) mainloop<KF32, KF64>(smem, full, empty, a, b, ksteps, acc);
  else if (a.kind == KF32) mainloop<KF32, KF32>(smem, full, empty, a, b, ksteps, acc);
  else if (b.kind == KF64) mainloop<KSPLIT, KF64>(smem, full, empty, a, b, ksteps, acc);
  else mainloop<KSPLIT, KSPLIT>(smem, full, empty, a, b, ksteps, acc);

  // epilogue: C fragment (row lane>>2, cols 2*(lane&3) + {0,1}) of each 8x8
  // block; all loads issued before any store
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;
  double* __restrict__ C = g.dtile(i, j);
  double2 cv[4][4];
#pragma unroll
  for (int fm = 0; fm < 4; ++fm)
#pragma unroll
    for (int fn = 0; fn < 4; ++fn)
      cv[fm][fn] = *(const double2*)(C + (int64_t)(m0 + wm + fm * 8 + (lane >> 2)) * nb + n0 +
                                     wn + fn * 8 + 2 * (lane & 3));
#pragma unroll
  for (int fm = 0; fm < 4; ++fm) {
    const int r = m0 + wm + fm * 8 + (lane >> 2);
#pragma unroll
    for (int fn = 0; fn < 4; ++fn) {
      const int c = n0 + wn + fn * 8 + 2 * (lane & 3);
      double2* cp = (double2*)(C + (int64_t)r * nb + c);
      const double2 v = make_double2(cv[fm][fn].x - acc[fm][fn][0], cv[fm][fn].y - acc[fm][fn][1]);
      if (!syrk || c + 1 <= r) *cp = v;
      else if (c <= r) C[(int64_t)r * nb + c] = v.x;
    }
  }
  if (span) {
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(&span[1], mt_globaltimer());
  }
}

}  // namespace

bool mt_dmma_tma_supported(const Grid& g) {
  return g.nb % BM == 0 && (int64_t)g.nband() * g.nb < (1ll << 31) &&
         (int64_t)g.noff() * g.nb < (1ll << 31) && (int64_t)4 * g.p * g.nb < (1ll << 31);
}

// band updates of step k into band slots [b0, b0 + bcnt).  pdl: launch as a
// programmatic dependent of the previous kernel on `st` (the capped bulk FP32
// update, which writes disjoint tiles): it starts on the SMs that update left
// free instead of after it.
int mt_dmma_update_impl(const Grid& g, int k, int64_t b0, int64_t bcnt, cudaStream_t st, bool pdl,
                        unsigned long long* span) {
  if (bcnt <= 0) return MT_OK;
  const int nb = g.nb;
  Maps maps;
  int rc = make_map_2d(&maps.dp, g.dp, g.nband() * nb, nb, 8, BK, 64, CU_TENSOR_MAP_SWIZZLE_128B);
  // maps that a layout does not use point at a valid dummy region (never loaded)
  const void* sp = g.sp ? (const void*)g.sp : (const void*)g.dp;
  const int64_t sp_rows = g.sp ? g.noff() * nb : nb;
  if (!rc) rc = make_map_2d(&maps.sp, sp, sp_rows, nb, 4, BK, 64, CU_TENSOR_MAP_SWIZZLE_64B);
  const void* spl = g.split ? (const void*)g.split : (const void*)g.dp;
  const int64_t spl_rows = g.split ? g.ring_rows() * nb : nb;
  if (!rc) rc = make_map_2d(&maps.split, spl, spl_rows, nb, 4, BK, 64, CU_TENSOR_MAP_SWIZZLE_64B);
  const void* dpn = g.dpanel ? (const void*)g.dpanel : (const void*)g.dp;
  const int64_t dpn_rows = g.dpanel ? (int64_t)g.nring * g.pring() * nb : nb;
  if (!rc) rc = make_map_2d(&maps.dpanel, dpn, dpn_rows, nb, 8, BK, 64, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  const int nsm = nb / BM, nsn = nb / BN;
  cudaFuncSetAttribute(dmma_tma_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  if (!pdl) {
    dmma_tma_update_kernel<<<(unsigned)(bcnt * nsm * nsn), 256, SMEM, st>>>(g, k, b0, nsm, nsn, maps,
                                                                             span);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(bcnt * nsm * nsn));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (mt_cuda_check(cudaLaunchKernelEx(&cfg, dmma_tma_update_kernel, g, k, b0, nsm, nsn, maps, span),
                      "dmma_tma_update_kernel (PDL)"))
      return MT_E_CUDA;
  }
  MT_LAUNCH_CHECK("dmma_tma_update_kernel");
  return MT_OK;
}
