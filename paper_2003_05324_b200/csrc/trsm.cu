// Panel TRSM of step k: A_ik <- A_ik L_kk^{-T} for every present i > k
// (kernels.trsm + factor.py:257-265), batched over the whole panel.
//
//   band rows    (i - k < t): FP64 against L_kk; in MP mode, when a later
//                FP32 update consumes the tile (i + t <= p - 1), the
//                epilogue also writes the RN-narrowed mirror (factor.py:261-262).
//   off-band rows (MP): FP32 against the narrowed L_kk (sp_diag,
//                factor.py:264); the FP64 view is the exact widening and is
//                never materialised (FP64 consumers widen on load).
//
// Rows of X = B L^{-T} are independent, so a CTA owns RB rows of one tile and
// walks the columns in 32-wide blocks: GEMM-style update from the solved
// columns (shared-memory X, streamed 32x32 chunks of L), then a warp-per-4-rows
// forward substitution on the 32x32 diagonal block with shuffle broadcasts.
#include "mt_grid.cuh"

namespace {

constexpr int kRB = 32;       // rows per CTA
constexpr int kThreads = 256; // 8 warps x 4 rows

template <typename T>
__global__ void __launch_bounds__(kThreads)
    trsm_kernel(Grid g, int k, int64_t slot0, int nrb, int mirror_ok) {
  if (g.failed()) return;
  const int64_t slot = slot0 + blockIdx.x / nrb;
  const int rb = blockIdx.x % nrb;
  int i, j;
  const T* L;
  T* B;
  float* M = nullptr;
  if constexpr (sizeof(T) == 8) {
    g.band_slot_ij(slot, i, j);
    L = (const T*)g.dtile(k, k);
    B = (T*)g.dtile(i, k);
    if (mirror_ok && g.mode == MT_MODE_MP && i + g.t <= g.p - 1) M = g.smirror(i, k);
  } else {
    g.off_slot_ij(slot, i, j);
    L = (const T*)g.sdiag(k);
    B = (T*)g.stile(i, k);
  }
  const int nb = g.nb;
  const int r0 = rb * kRB;
  const int nr = min(kRB, nb - r0);
  extern __shared__ unsigned char smem_raw[];
  T* X = (T*)smem_raw;                 // kRB x (nb + 1)
  T* Lc = X + kRB * (nb + 1);          // 32 x 33 chunk of L
  const int ldx = nb + 1;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int row0 = warp * 4;  // this warp's 4 rows (local)

  for (int cb = 0; cb < nb; cb += 32) {
    const int w = min(32, nb - cb);
    T acc[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int r = row0 + a;
      acc[a] = (r < nr && lane < w) ? B[(int64_t)(r0 + r) * nb + cb + lane] : T(0);
    }
    // acc[r][c] -= sum_{q < cb} X[r][q] L[cb + c][q]
    for (int q0 = 0; q0 < cb; q0 += 32) {
      __syncthreads();
      for (int e = threadIdx.x; e < 32 * 32; e += kThreads) {
        int rr = e >> 5, cc = e & 31;
        Lc[rr * 33 + cc] = (rr < w) ? L[(int64_t)(cb + rr) * nb + q0 + cc] : T(0);
      }
      __syncthreads();
#pragma unroll 8
      for (int q = 0; q < 32; ++q) {
        T l = Lc[lane * 33 + q];
#pragma unroll
        for (int a = 0; a < 4; ++a) acc[a] -= X[(row0 + a) * ldx + q0 + q] * l;
      }
    }
    // diagonal block L[cb:cb+w, cb:cb+w]
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * 32; e += kThreads) {
      int rr = e >> 5, cc = e & 31;
      Lc[rr * 33 + cc] = (rr < w && cc < w) ? L[(int64_t)(cb + rr) * nb + cb + cc] : T(0);
    }
    __syncthreads();
    for (int c = 0; c < w; ++c) {
      const T dcc = Lc[c * 33 + c];
      const T lc = Lc[lane * 33 + c];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        T xc = __shfl_sync(0xffffffffu, acc[a], c) / dcc;
        if (lane == c) acc[a] = xc;
        else if (lane > c) acc[a] -= xc * lc;
      }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int r = row0 + a;
      if (lane < w) X[r * ldx + cb + lane] = acc[a];
    }
  }
  __syncthreads();
  // write back; FP32 operands of this step's FP32 updates also get their
  // narrowed mirror (band rows, factor.py:261-262) and, for the tensor-core
  // engine, the TF32 hi/lo split (hi = rna(x), lo = x - hi) read by UMMA
  const bool fp32_operand = (sizeof(T) == 4) || (M != nullptr);
  float* SH = (g.split && fp32_operand) ? g.split_hi(i, k) : nullptr;
  float* SL = SH ? g.split_lo(i, k) : nullptr;
  for (int e = threadIdx.x; e < nr * nb; e += kThreads) {
    int r = e / nb, c = e % nb;
    T v = X[r * ldx + c];
    const int64_t o = (int64_t)(r0 + r) * nb + c;
    B[o] = v;
    const float f = __double2float_rn((double)v);
    if (M) M[o] = f;
    if (SH) {
      uint32_t h;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(f));
      SH[o] = __uint_as_float(h);
      SL[o] = f - __uint_as_float(h);
    }
  }
}

template <typename T>
int launch_trsm(const Grid& g, int k, int64_t s0, int64_t cnt, int mirror_ok, cudaStream_t st) {
  if (cnt <= 0) return MT_OK;
  const int nrb = (g.nb + kRB - 1) / kRB;
  size_t smem = ((size_t)kRB * (g.nb + 1) + 32 * 33) * sizeof(T);
  cudaFuncSetAttribute(trsm_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  const double rk = g.rows(k), nb = g.nb;
  // algorithmic work: rows(i) * rows(k)^2 per tile (factor.py:88-90); last row may be ragged
  const bool last = (sizeof(T) == 8 ? (k + g.t >= g.p) : true) && cnt > 0;
  const double rows_sum = (cnt - (last ? 1 : 0)) * nb + (last ? g.rows(g.p - 1) : 0);
  ProfScope ps(sizeof(T) == 8 ? MT_K_TRSM64 : MT_K_TRSM32, st, rows_sum * rk * rk,
               cnt * nb * nb * sizeof(T) * 2.0);
  trsm_kernel<T><<<(unsigned)(cnt * nrb), kThreads, smem, st>>>(g, k, s0, nrb, mirror_ok);
  MT_LAUNCH_CHECK("trsm_kernel");
  return MT_OK;
}

}  // namespace

// Panel rows i in (k, p) of tile column k.  Band rows: band slots
// bcol(k)+1 .. bcol(k+1)-1; off-band rows: off slots scol(k) .. scol(k+1)-1.
int mt_trsm_impl(const Grid& g, int k, cudaStream_t st) {
  if ((size_t)32 * (g.nb + 1) * sizeof(double) > 200 * 1024) {
    mt_set_error("trsm: nb=%d too large for the shared-memory panel", g.nb);
    return MT_E_BAD_ARG;
  }
  int rc = launch_trsm<double>(g, k, g.bcol(k) + 1, g.bcol(k + 1) - g.bcol(k) - 1, 1, st);
  if (rc) return rc;
  if (g.mode == MT_MODE_MP) rc = launch_trsm<float>(g, k, g.scol(k), g.scol(k + 1) - g.scol(k), 0, st);
  return rc;
}
