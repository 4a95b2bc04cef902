// Diagonal-tile Cholesky POTRF(k), FP64, in place on the row-major tile
// (kernels.potrf + factor.py:249-256).
//
// One CTA of 512 threads walks the tile in BW-wide column blocks
// (right-looking): warp 0 factors the BW x BW diagonal block in shared
// memory, all warps solve the sub-diagonal panel (warp per row, lane per
// column, shuffle broadcast), then the trailing lower triangle takes a rank-BW
// SYRK update from the shared-memory panel with 4x4 register blocks.
// Epilogue: the first non-positive (or NaN) pivot is published as the global
// index k*nb + j (FactorizationError.index), and in MP mode the factored
// tile is narrowed to FP32 scratch for the off-band panel solves (sp_diag,
// factor.py:255-256).  The strict upper triangle is never written.
#include "mt_grid.cuh"

namespace {

constexpr int kThreads = 512;

template <int BW>
__global__ void __launch_bounds__(kThreads) potrf_kernel(Grid g, int k, int narrow) {
  if (g.failed()) return;
  double* __restrict__ A = g.dtile(k, k);
  const int nb = g.nb;
  __shared__ double Ld[BW][BW + 1];
  __shared__ int bad;
  extern __shared__ double P[];  // (nb - BW) x (BW + 1) panel
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  constexpr int nwarps = kThreads / 32;
  if (threadIdx.x == 0) bad = -1;

  for (int c0 = 0; c0 < nb; c0 += BW) {
    const int w = min(BW, nb - c0);
    for (int e = threadIdx.x; e < w * w; e += kThreads) {
      int r = e / w, c = e % w;
      if (c <= r) Ld[r][c] = A[(int64_t)(c0 + r) * nb + c0 + c];
    }
    __syncthreads();
    // --- factor the diagonal block (warp 0, lane r owns row r) ---
    if (warp == 0) {
      for (int jj = 0; jj < w; ++jj) {
        double piv = Ld[jj][jj];
        if (!(piv > 0.0)) {
          if (lane == 0) bad = c0 + jj;
          break;
        }
        double d = sqrt(piv);
        __syncwarp();
        if (lane > jj && lane < w) Ld[lane][jj] = Ld[lane][jj] / d;
        if (lane == jj) Ld[jj][jj] = d;
        __syncwarp();
        if (lane > jj && lane < w) {
          double lr = Ld[lane][jj];
          for (int l = jj + 1; l <= lane; ++l) Ld[lane][l] -= lr * Ld[l][jj];
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (bad >= 0) {
      if (threadIdx.x == 0)
        atomicCAS((unsigned long long*)&g.status[MT_ST_PIVOT], (unsigned long long)-1LL,
                  (unsigned long long)((int64_t)k * nb + bad));
      return;
    }
    for (int e = threadIdx.x; e < w * w; e += kThreads) {
      int r = e / w, c = e % w;
      if (c <= r) A[(int64_t)(c0 + r) * nb + c0 + c] = Ld[r][c];
    }
    // --- panel solve: rows below the block, x <- a L_dd^{-T} ---
    const int r_lo = c0 + w;
    for (int r = r_lo + warp; r < nb; r += nwarps) {
      double acc = lane < w ? A[(int64_t)r * nb + c0 + lane] : 0.0;
      for (int c = 0; c < w; ++c) {
        double xc = __shfl_sync(0xffffffffu, acc, c) / Ld[c][c];
        if (lane == c) acc = xc;
        else if (lane > c && lane < w) acc -= xc * Ld[lane][c];
      }
      if (lane < w) {
        A[(int64_t)r * nb + c0 + lane] = acc;
        P[(r - r_lo) * (BW + 1) + lane] = acc;
      }
    }
    __syncthreads();
    // --- trailing SYRK: A[r][c] -= P[r] . P[c], r >= c >= r_lo ---
    const int m = nb - r_lo;
    if (m > 0) {
      const int nblk = (m + 3) / 4;
      const int ntri = nblk * (nblk + 1) / 2;
      for (int L = threadIdx.x; L < ntri; L += kThreads) {
        int br = (int)((sqrtf(8.0f * (float)L + 1.0f) - 1.0f) * 0.5f);
        while (br * (br + 1) / 2 > L) --br;
        while ((br + 1) * (br + 2) / 2 <= L) ++br;
        const int bc = L - br * (br + 1) / 2;
        double acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
        int rr[4], cc[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          rr[a] = min(br * 4 + a, m - 1);
          cc[a] = min(bc * 4 + a, m - 1);
        }
        for (int q = 0; q < w; ++q) {
          double pa[4], pb[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            pa[a] = P[rr[a] * (BW + 1) + q];
            pb[a] = P[cc[a] * (BW + 1) + q];
          }
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] += pa[a] * pb[b];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int r = br * 4 + a;
          if (r >= m) continue;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int c = bc * 4 + b;
            if (c < m && c <= r) A[(int64_t)(r_lo + r) * nb + r_lo + c] -= acc[a][b];
          }
        }
      }
    }
    __syncthreads();
  }
  if (narrow) {
    float* S = g.sdiag(k);
    const int64_t tot = (int64_t)nb * nb;
    for (int64_t e = threadIdx.x; e < tot; e += kThreads) {
      int r = (int)(e / nb), c = (int)(e % nb);
      S[e] = c <= r ? __double2float_rn(A[e]) : 0.0f;
    }
  }
}

template <int BW>
int launch_potrf(const Grid& g, int k, int narrow, cudaStream_t st) {
  size_t smem = (size_t)(g.nb > BW ? g.nb - BW : 1) * (BW + 1) * sizeof(double);
  cudaFuncSetAttribute(potrf_kernel<BW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       200 * 1024);
  const double r = g.rows(k);
  ProfScope ps(MT_K_POTRF, st, r * r * r / 3.0, (double)g.nb * g.nb * (16.0 + (narrow ? 4.0 : 0.0)));
  potrf_kernel<BW><<<1, kThreads, smem, st>>>(g, k, narrow);
  MT_LAUNCH_CHECK("potrf_kernel");
  return MT_OK;
}

}  // namespace

int mt_potrf_impl(const Grid& g, int k, int narrow, cudaStream_t st) {
  if (g.nb <= 704) return launch_potrf<32>(g, k, narrow, st);
  if (g.nb <= 1408) return launch_potrf<16>(g, k, narrow, st);
  mt_set_error("potrf: nb=%d exceeds the supported maximum 1408", g.nb);
  return MT_E_BAD_ARG;
}
