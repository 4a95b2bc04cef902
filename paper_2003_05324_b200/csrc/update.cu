// Trailing update of step k over tile columns [jlo, jhi):
//   C_ij <- C_ij - A_ik A_jk^T   for k < j <= i < p   (kernels.syrk / kernels.gemm,
//                                                     factor.py:266-274)
// Band outputs (i - j < t) run in FP64; an off-band operand (FP32 payload) is
// widened in registers on load, which is bit-identical to the reference's
// materialised widened copy (factor.py:265, test_factor.py:146-153).  SYRK
// outputs (i == j) touch the lower triangle only.  Off-band outputs (MP)
// run in FP32 against the FP32 payload / narrowed band mirror.
//
// Each output tile's updates are applied by exactly one CTA per sub-tile and
// step, in ascending k -- no split-K, no atomics -- so results are
// deterministic and schedule-invariant (factor.py:13-16).
#include "mt_grid.cuh"

namespace {

// ---------------------------------------------------------------- FP32 SIMT
// 128x128 CTA tile, BK=8, 256 threads x (8x8) outputs, register double buffering.
constexpr int SBM = 128, SBK = 8;

__global__ void __launch_bounds__(256)
    sgemm_update_kernel(Grid g, int k, int64_t slot0, int nsub) {
  if (g.failed()) return;
  const int64_t slot = slot0 + blockIdx.x / (nsub * nsub);
  const int sub = blockIdx.x % (nsub * nsub);
  int i, j;
  g.off_slot_ij(slot, i, j);
  const int nb = g.nb;
  const int m0 = (sub / nsub) * SBM, n0 = (sub % nsub) * SBM;
  const float* __restrict__ A = g.stile(i, k) + (int64_t)m0 * nb;
  const float* __restrict__ B = g.sp_operand(j, k) + (int64_t)n0 * nb;
  float* __restrict__ C = g.stile(i, j);

  __shared__ __align__(16) float As[2][SBK][SBM];
  __shared__ __align__(16) float Bs[2][SBK][SBM];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int lr = tid >> 1, lc = (tid & 1) * 4;  // load: row lr, cols lc..lc+3

  float acc[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = 0.f;

  float4 ra = *(const float4*)(A + (int64_t)lr * nb + lc);
  float4 rb = *(const float4*)(B + (int64_t)lr * nb + lc);
  As[0][lc + 0][lr] = ra.x; As[0][lc + 1][lr] = ra.y; As[0][lc + 2][lr] = ra.z; As[0][lc + 3][lr] = ra.w;
  Bs[0][lc + 0][lr] = rb.x; Bs[0][lc + 1][lr] = rb.y; Bs[0][lc + 2][lr] = rb.z; Bs[0][lc + 3][lr] = rb.w;
  __syncthreads();
  int buf = 0;
  for (int kk = 0; kk < nb; kk += SBK) {
    const bool more = kk + SBK < nb;
    if (more) {
      ra = *(const float4*)(A + (int64_t)lr * nb + kk + SBK + lc);
      rb = *(const float4*)(B + (int64_t)lr * nb + kk + SBK + lc);
    }
#pragma unroll
    for (int q = 0; q < SBK; ++q) {
      float4 a0 = *(const float4*)&As[buf][q][ty * 4];
      float4 a1 = *(const float4*)&As[buf][q][64 + ty * 4];
      float4 b0 = *(const float4*)&Bs[buf][q][tx * 4];
      float4 b1 = *(const float4*)&Bs[buf][q][64 + tx * 4];
      float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = fmaf(av[a], bv[b], acc[a][b]);
    }
    if (more) {
      const int nbuf = buf ^ 1;
      As[nbuf][lc + 0][lr] = ra.x; As[nbuf][lc + 1][lr] = ra.y; As[nbuf][lc + 2][lr] = ra.z; As[nbuf][lc + 3][lr] = ra.w;
      Bs[nbuf][lc + 0][lr] = rb.x; Bs[nbuf][lc + 1][lr] = rb.y; Bs[nbuf][lc + 2][lr] = rb.z; Bs[nbuf][lc + 3][lr] = rb.w;
      __syncthreads();
      buf = nbuf;
    }
  }
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int r = m0 + (a < 4 ? ty * 4 + a : 64 + ty * 4 + a - 4);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float4* cp = (float4*)(C + (int64_t)r * nb + n0 + h * 64 + tx * 4);
      float4 c = *cp;
      c.x -= acc[a][h * 4 + 0];
      c.y -= acc[a][h * 4 + 1];
      c.z -= acc[a][h * 4 + 2];
      c.w -= acc[a][h * 4 + 3];
      *cp = c;
    }
  }
}

// ---------------------------------------------------------------- FP64 SIMT
// 64x64 CTA tile, BK=8, 256 threads x (4x4); operands FP64 or FP32 (widened).
constexpr int DBM = 64, DBK = 8;

__device__ __forceinline__ double2 ld2(const void* base, bool f32, int64_t idx) {
  if (f32) {
    float2 v = *(const float2*)((const float*)base + idx);
    return make_double2((double)v.x, (double)v.y);
  }
  return *(const double2*)((const double*)base + idx);
}

__global__ void __launch_bounds__(256)
    dgemm_update_kernel(Grid g, int k, int64_t slot0, int nsub) {
  if (g.failed()) return;
  const int64_t slot = slot0 + blockIdx.x / (nsub * nsub);
  const int sub = blockIdx.x % (nsub * nsub);
  int i, j;
  g.band_slot_ij(slot, i, j);
  if (!g.present(i, k)) return;  // DST: GEMM(k; i, j) needs tile (i, k)
  const int bm = sub / nsub, bn = sub % nsub;
  const bool syrk = (i == j);
  if (syrk && bn > bm) return;  // strict upper sub-tiles of a diagonal tile
  const int nb = g.nb;
  const int m0 = bm * DBM, n0 = bn * DBM;
  const bool fa = !g.band(i, k), fb = !g.band(j, k);
  const void* A = fa ? (const void*)g.stile(i, k) : (const void*)g.dtile(i, k);
  const void* B = fb ? (const void*)g.stile(j, k) : (const void*)g.dtile(j, k);
  double* __restrict__ C = g.dtile(i, j);

  __shared__ __align__(16) double As[2][DBK][DBM + 2];
  __shared__ __align__(16) double Bs[2][DBK][DBM + 2];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int lr = tid >> 2, lc = (tid & 3) * 2;

  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;

  const int64_t arow = (int64_t)(m0 + lr) * nb, brow = (int64_t)(n0 + lr) * nb;
  double2 ra = ld2(A, fa, arow + lc), rb = ld2(B, fb, brow + lc);
  As[0][lc][lr] = ra.x; As[0][lc + 1][lr] = ra.y;
  Bs[0][lc][lr] = rb.x; Bs[0][lc + 1][lr] = rb.y;
  __syncthreads();
  int buf = 0;
  for (int kk = 0; kk < nb; kk += DBK) {
    const bool more = kk + DBK < nb;
    if (more) {
      ra = ld2(A, fa, arow + kk + DBK + lc);
      rb = ld2(B, fb, brow + kk + DBK + lc);
    }
#pragma unroll
    for (int q = 0; q < DBK; ++q) {
      double2 a0 = *(const double2*)&As[buf][q][ty * 4];
      double2 a1 = *(const double2*)&As[buf][q][ty * 4 + 2];
      double2 b0 = *(const double2*)&Bs[buf][q][tx * 4];
      double2 b1 = *(const double2*)&Bs[buf][q][tx * 4 + 2];
      double av[4] = {a0.x, a0.y, a1.x, a1.y};
      double bv[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
    }
    if (more) {
      const int nbuf = buf ^ 1;
      As[nbuf][lc][lr] = ra.x; As[nbuf][lc + 1][lr] = ra.y;
      Bs[nbuf][lc][lr] = rb.x; Bs[nbuf][lc + 1][lr] = rb.y;
      __syncthreads();
      buf = nbuf;
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int r = m0 + ty * 4 + a;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int c = n0 + tx * 4 + b;
      if (!syrk || c <= r) C[(int64_t)r * nb + c] -= acc[a][b];
    }
  }
}

// ---------------------------------------------------------------- FP64 DMMA
// 128x64 CTA tile, 8 warps x (32x32) warp tiles of m8n8k4 f64 MMAs (SASS DMMA);
// operands FP64 or FP32 (widened on load), register-prefetched one K slab
// ahead, smem rows padded to 20 doubles (conflict-free fragment loads).
constexpr int MBM = 128, MBN = 64, MBK = 16, MLD = MBK + 4;
constexpr int MMA_SMEM = 2 * (MBM + MBN) * MLD * 8;

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// FP64 view of an operand tile of panel k: FP64 payload, FP32 payload (widened),
// or -- on a multi-GPU rank that received the panel -- the TF32 split hi + lo,
// whose FP64 sum is exactly the FP32 payload (lo = x - hi is exact in FP32)
struct Operand {
  const void* base;
  const float* lo;  // non-null: hi/lo split
  bool f32;
};
__device__ __forceinline__ Operand panel_operand(const Grid& g, int i, int k) {
  Operand o;
  o.lo = nullptr;
  if (g.band(i, k)) {
    o.base = !g.multi() ? (const void*)g.dtile(i, k) : (const void*)g.dpanel_tile(i, k);
    o.f32 = false;
  } else if (!g.multi()) {
    o.base = g.stile(i, k);
    o.f32 = true;
  } else {
    o.base = g.split_hi(i, k);
    o.lo = g.split_lo(i, k);
    o.f32 = true;
  }
  return o;
}

// 8 consecutive operand values starting at idx, as FP64
__device__ __forceinline__ void ld8(const Operand& o, int64_t idx, double (&v)[8]) {
  if (o.f32) {
    const float4* p = (const float4*)((const float*)o.base + idx);
    float4 x = p[0], y = p[1];
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w; v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
    if (o.lo) {
      const float4* q = (const float4*)(o.lo + idx);
      float4 a = q[0], b = q[1];
      v[0] += a.x; v[1] += a.y; v[2] += a.z; v[3] += a.w;
      v[4] += b.x; v[5] += b.y; v[6] += b.z; v[7] += b.w;
    }
  } else {
    const double2* p = (const double2*)((const double*)o.base + idx);
#pragma unroll
    for (int q = 0; q < 4; ++q) { double2 t = p[q]; v[2 * q] = t.x; v[2 * q + 1] = t.y; }
  }
}
__device__ __forceinline__ void ld4(const Operand& o, int64_t idx, double (&v)[4]) {
  if (o.f32) {
    float4 x = *(const float4*)((const float*)o.base + idx);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    if (o.lo) {
      float4 a = *(const float4*)(o.lo + idx);
      v[0] += a.x; v[1] += a.y; v[2] += a.z; v[3] += a.w;
    }
  } else {
    const double2* p = (const double2*)((const double*)o.base + idx);
    double2 s = p[0], t = p[1];
    v[0] = s.x; v[1] = s.y; v[2] = t.x; v[3] = t.y;
  }
}

__global__ void __launch_bounds__(256, 2)
    dmma_update_kernel(Grid g, int k, int64_t slot0, int nsubm, int nsubn) {
  if (g.failed()) return;
  const int nsub = nsubm * nsubn;
  const int64_t slot = slot0 + blockIdx.x / nsub;
  const int sub = blockIdx.x % nsub;
  int i, j;
  g.band_slot_ij(slot, i, j);
  if (!g.present(i, k)) return;  // DST: GEMM(k; i, j) needs tile (i, k)
  const int m0 = (sub / nsubn) * MBM, n0 = (sub % nsubn) * MBN;
  const bool syrk = (i == j);
  if (syrk && n0 >= m0 + MBM) return;  // entirely above the diagonal
  const int nb = g.nb;
  const Operand A = panel_operand(g, i, k), B = panel_operand(g, j, k);
  double* __restrict__ C = g.dtile(i, j);

  extern __shared__ __align__(16) double msm[];
  double* As = msm;                      // [2][MBM][MLD]
  double* Bs = msm + 2 * MBM * MLD;      // [2][MBN][MLD]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;
  const int ar = tid >> 1, ac = (tid & 1) * 8;   // A slab: 128 rows x 16
  const int br = tid >> 2, bc = (tid & 3) * 4;   // B slab:  64 rows x 16
  const int64_t abase = (int64_t)(m0 + ar) * nb + ac, bbase = (int64_t)(n0 + br) * nb + bc;

  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  double ra[8], rb[4];
  ld8(A, abase, ra);
  ld4(B, bbase, rb);
  int buf = 0;
  for (int kk = 0; kk < nb; kk += MBK) {
    double* as = As + buf * MBM * MLD;
    double* bs = Bs + buf * MBN * MLD;
#pragma unroll
    for (int q = 0; q < 4; ++q) *(double2*)&as[ar * MLD + ac + 2 * q] = make_double2(ra[2 * q], ra[2 * q + 1]);
    *(double2*)&bs[br * MLD + bc] = make_double2(rb[0], rb[1]);
    *(double2*)&bs[br * MLD + bc + 2] = make_double2(rb[2], rb[3]);
    __syncthreads();
    if (kk + MBK < nb) {
      ld8(A, abase + kk + MBK, ra);
      ld4(B, bbase + kk + MBK, rb);
    }
#pragma unroll
    for (int k4 = 0; k4 < MBK; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        af[f] = as[(wm + f * 8 + (lane >> 2)) * MLD + k4 + (lane & 3)];
        bf[f] = bs[(wn + f * 8 + (lane >> 2)) * MLD + k4 + (lane & 3)];
      }
#pragma unroll
      for (int fm = 0; fm < 4; ++fm)
#pragma unroll
        for (int fn = 0; fn < 4; ++fn) dmma884(acc[fm][fn], af[fm], bf[fn]);
    }
    buf ^= 1;
  }
  // epilogue: C fragment (row lane>>2, cols 2*(lane&3) + {0,1}) of each 8x8
  // block; all loads are issued before any store (no load/store serialisation)
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
}

// ------------------------------------------------- generic (any nb) fallback
template <bool F64>
__global__ void __launch_bounds__(256)
    gemm_generic_kernel(Grid g, int k, int64_t slot0, int nblk) {
  if (g.failed()) return;
  const int64_t slot = slot0 + blockIdx.x / nblk;
  const int64_t e = (int64_t)(blockIdx.x % nblk) * 256 + threadIdx.x;
  const int nb = g.nb;
  if (e >= (int64_t)nb * nb) return;
  const int r = (int)(e / nb), c = (int)(e % nb);
  int i, j;
  if (F64) {
    g.band_slot_ij(slot, i, j);
    if (!g.present(i, k)) return;
    if (i == j && c > r) return;
    const bool fa = !g.band(i, k), fb = !g.band(j, k);
    double acc = 0.0;
    for (int q = 0; q < nb; ++q) {
      double a = fa ? (double)g.stile(i, k)[(int64_t)r * nb + q] : g.dtile(i, k)[(int64_t)r * nb + q];
      double b = fb ? (double)g.stile(j, k)[(int64_t)c * nb + q] : g.dtile(j, k)[(int64_t)c * nb + q];
      acc = fma(a, b, acc);
    }
    g.dtile(i, j)[e] -= acc;
  } else {
    g.off_slot_ij(slot, i, j);
    const float* A = g.stile(i, k);
    const float* B = g.sp_operand(j, k);
    float acc = 0.f;
    for (int q = 0; q < nb; ++q) acc = fmaf(A[(int64_t)r * nb + q], B[(int64_t)c * nb + q], acc);
    g.stile(i, j)[e] -= acc;
  }
}

}  // namespace

// algorithmic flops of step k's updates into columns [jlo, jhi) (factor.py:91-95)
static void update_flops(const Grid& g, int k, int jlo, int jhi, double& f64, double& f32) {
  f64 = f32 = 0.0;
  const double rk = g.rows(k);
  for (int j = jlo; j < jhi; ++j) {
    if (!g.owns_col(j)) continue;  // (rows: only this rank's, below)
    const double rj = g.rows(j);
    const int iband = j + g.t < g.p ? j + g.t : g.p;  // band rows [j, iband)
    for (int i = j; i < iband; ++i) {
      if (!g.present(i, k) || !g.owns_row(i)) continue;
      const double ri = g.rows(i);
      f64 += (i == j) ? ri * ri * rk : 2.0 * ri * rj * rk;
    }
    if (g.mode == MT_MODE_MP && iband < g.p) {  // off-band rows [iband, p): last may be ragged
      const double cnt = g.rcnt(g.p) - g.rcnt(iband);
      if (cnt > 0) {
        const double last = g.owns_row(g.p - 1) ? g.rows(g.p - 1) : g.nb;
        f32 += 2.0 * rj * rk * ((cnt - 1) * g.nb + last);
      }
    }
  }
}

#define RC_UPD(call) \
  do { int rc__ = (call); if (rc__) return rc__; } while (0)

int mt_update_impl(const Grid& g, int k, int jlo, int jhi, cudaStream_t st) {
  if (jlo >= jhi) return MT_OK;
  const int nb = g.nb;
  if (g.multi() && (nb % MBM != 0 || (g.mode == MT_MODE_MP && !mt_tc_supported(g)))) {
    mt_set_error("multi-GPU layout needs nb %% 256 == 0 and the tcgen05 engine (split buffer)");
    return MT_E_BAD_ARG;
  }
  double f64, f32;
  update_flops(g, k, jlo, jhi, f64, f32);
  const bool pcol = (jlo == k + 1 && jhi == jlo + 1 && jhi < g.p);  // lookahead panel column
  // Co-scheduling (option 10): the bulk FP32 update runs on a capped set of
  // SM pairs and the FP64 band update is launched as its programmatic
  // dependent, filling the remaining SMs -- DMMA work (low power) then runs
  // beside the power-capped tensor-core work instead of after it.  The split
  // follows the step's FP64/FP32 work at the measured pipe rates; the band
  // update gets slightly less than its share so it, not the capped FP32
  // update, absorbs the tail (its CTAs spread onto the SMs the update frees).
  const int64_t co_s0 = g.scol(jlo), co_scnt = g.scol(jhi) - co_s0;
  const int64_t co_b0 = g.bcol(jlo), co_bcnt = g.bcol(jhi) - co_b0;
  if (mt_opt_coschedule() && !pcol && g.mode == MT_MODE_MP && co_scnt > 0 && co_bcnt > 0 &&
      (mt_engine_tc(mt_opt_engine()) || g.multi()) && mt_tc_supported(g) &&
      mt_opt_legacy_dmma() != 1 && mt_dmma_tma_supported(g)) {
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const double a = f64 / 32e12, b = f32 / 215e12;  // seconds on the whole GPU
    int x = (int)(0.01 * mt_opt_coschedule_pct() * sms * a / (a + b));  // SMs left to the band update
    if (x > sms - 2) x = sms - 2;
    int tc_ctas = (sms - x) & ~1;
    if (tc_ctas < 2) tc_ctas = 2;
    // no stream events between the two launches (they would serialise them):
    // both kernels stamp device-side spans for the profiler
    mt_count_launch(2);
    unsigned long long* s32 = mt_prof_dspan(MT_K_UPD32, f32, co_scnt * (double)nb * nb * 4.0 * 2.0,
                                            (double)tc_ctas / sms);
    unsigned long long* s64 = mt_prof_dspan(MT_K_UPD64, f64, co_bcnt * (double)nb * nb * 8.0 * 3.0);
    RC_UPD(mt_tc_update_impl(g, k, jlo, jhi, tc_ctas, st, s32));
    return mt_dmma_update_impl(g, k, co_b0, co_bcnt, st, true, s64);
  }
  // band (FP64) outputs in columns [jlo, jhi)
  const int64_t b0 = g.bcol(jlo), bcnt = g.bcol(jhi) - b0;
  if (bcnt > 0) {
    int return_rc = MT_OK;
    ProfScope ps(pcol ? MT_K_UPD64P : MT_K_UPD64, st, f64, bcnt * (double)nb * nb * 8.0 * 3.0);
    if (mt_opt_legacy_dmma() != 1 && mt_dmma_tma_supported(g)) {
      return_rc = mt_dmma_update_impl(g, k, b0, bcnt, st);
    } else if (nb % MBM == 0) {
      const int nsm = nb / MBM, nsn = nb / MBN;
      cudaFuncSetAttribute(dmma_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           MMA_SMEM);
      dmma_update_kernel<<<(unsigned)(bcnt * nsm * nsn), 256, MMA_SMEM, st>>>(g, k, b0, nsm, nsn);
    } else if (nb % DBM == 0) {
      const int nsub = nb / DBM;
      dgemm_update_kernel<<<(unsigned)(bcnt * nsub * nsub), 256, 0, st>>>(g, k, b0, nsub);
    } else {
      const int nblk = (nb * nb + 255) / 256;
      gemm_generic_kernel<true><<<(unsigned)(bcnt * nblk), 256, 0, st>>>(g, k, b0, nblk);
    }
    if (return_rc) return return_rc;
    MT_LAUNCH_CHECK("dgemm_update");
  }
  if (g.mode != MT_MODE_MP) return MT_OK;
  const int64_t s0 = g.scol(jlo), scnt = g.scol(jhi) - s0;
  if (scnt > 0) {
    ProfScope ps(pcol ? MT_K_UPD32P : MT_K_UPD32, st, f32, scnt * (double)nb * nb * 4.0 * 2.0);
    if ((mt_engine_tc(mt_opt_engine()) || g.multi()) && mt_tc_supported(g)) {
      // the panel-column update (jhi == jlo + 1) runs beside the bulk update:
      // keep it narrow; the bulk update may be capped to leave SMs for the panel
      const int ctas = (jhi == jlo + 1) ? mt_opt_pcol_ctas() : mt_opt_update_ctas();
      return mt_tc_update_impl(g, k, jlo, jhi, ctas, st);
    }
    if (nb % SBM == 0) {
      const int nsub = nb / SBM;
      sgemm_update_kernel<<<(unsigned)(scnt * nsub * nsub), 256, 0, st>>>(g, k, s0, nsub);
    } else {
      const int nblk = (nb * nb + 255) / 256;
      gemm_generic_kernel<false><<<(unsigned)(scnt * nblk), 256, 0, st>>>(g, k, s0, nblk);
    }
    MT_LAUNCH_CHECK("sgemm_update");
  }
  return MT_OK;
}
