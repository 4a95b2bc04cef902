// Operations on the factor (factor.py:292-340, mle.py:80-86), all FP64.
//
//   logdet      2 sum_k sum_r log L_kk[r][r]: one CTA per diagonal tile with a
//               fixed-order tree reduction, then a fixed-order sum over k.
//   forward     L y = b by tile columns: diagonal-tile TRSV (one CTA, 32-row
//               blocks, warp-shuffle substitution) then the column-panel GEMV
//               b_r -= L_ri y_i over every present r > i (one launch).
//   backward    L^T x = y by tile rows: diagonal TRSV^T, then x_j -= L_ij^T x_i
//               for j < i.
//   quad        ||L^{-1} z||^2 after the forward sweep only (= z^T Sigma^{-1} z).
//   matvec      L v (generate_field's Z = L v, geodata.py:88-106).
// Off-band tiles are read as FP32 and widened (their FP64 view is exactly the
// widening, factor.py:264-265); DST tiles that are absent are skipped.
// No atomics: every output element has one writer and a fixed summation order.
#include "mt_grid.cuh"

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// element (r, c) of tile (i, j) as FP64; false if the tile is absent
struct TileRef {
  const double* d;
  const float* f;
  __device__ __forceinline__ double at(int64_t e) const { return d ? d[e] : (double)f[e]; }
};
__device__ __forceinline__ bool tile_ref(const Grid& g, int i, int j, TileRef& t) {
  if (!g.present(i, j)) return false;
  if (g.band(i, j)) { t.d = g.dtile(i, j); t.f = nullptr; }
  else { t.d = nullptr; t.f = g.stile(i, j); }
  return true;
}

// ------------------------------------------------------------------ logdet
__global__ void __launch_bounds__(256) logdet_partial_kernel(Grid g, double* partial) {
  const int k = blockIdx.x;
  if (!g.owns(k, k)) {  // multi-GPU: another rank holds this diagonal tile
    if (threadIdx.x == 0) partial[k] = 0.0;
    return;
  }
  const double* L = g.dtile(k, k);
  const int nb = g.nb;
  double s = 0.0;
  for (int r = threadIdx.x; r < nb; r += blockDim.x) s += log(L[(int64_t)r * nb + r]);
  __shared__ double red[8];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    partial[k] = t;
  }
}

__global__ void fixed_sum_kernel(const double* v, int m, double scale, double* out) {
  double t = 0.0;
  for (int q = 0; q < m; ++q) t += v[q];
  *out = scale * t;
}

// ----------------------------------------------------------- forward sweep
// y_i = L_ii^{-1} x_i in place, one CTA (512 threads), per right-hand side.
__global__ void __launch_bounds__(512) trsv_fwd_diag_kernel(Grid g, int i, double* x,
                                                            int64_t nrhs) {
  const double* L = g.dtile(i, i);
  const int nb = g.nb;
  extern __shared__ double ys[];  // nb
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t c = 0; c < nrhs; ++c) {
    double* xi = x + (int64_t)i * nb * nrhs + c;
    for (int r = threadIdx.x; r < nb; r += blockDim.x) ys[r] = xi[(int64_t)r * nrhs];
    __syncthreads();
    for (int cb = 0; cb < nb; cb += 32) {
      const int w = min(32, nb - cb);
      // rows cb..cb+w-1: ys[r] -= L[r][0:cb] . ys[0:cb]   (warp per row)
      if (cb > 0) {
        for (int rr = warp; rr < w; rr += blockDim.x >> 5) {
          const int r = cb + rr;
          double s = 0.0;
          for (int q = lane; q < cb; q += 32) s += L[(int64_t)r * nb + q] * ys[q];
          s = warp_sum(s);
          if (lane == 0) ys[r] -= s;
        }
        __syncthreads();
      }
      if (warp == 0) {
        // stage the 32x32 diagonal block: lane r keeps row r in registers,
        // so the serial substitution never waits on global memory
        double lr[32];
#pragma unroll
        for (int q = 0; q < 32; ++q)
          lr[q] = (lane < w && q < w) ? L[(int64_t)(cb + lane) * nb + cb + q] : 1.0;
        double acc = lane < w ? ys[cb + lane] : 0.0;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          if (q < w) {
            const double dq = __shfl_sync(0xffffffffu, lr[q], q);
            const double yq = __shfl_sync(0xffffffffu, acc, q) / dq;
            if (lane == q) acc = yq;
            else if (lane > q && lane < w) acc -= lr[q] * yq;
          }
        }
        if (lane < w) ys[cb + lane] = acc;
      }
      __syncthreads();
    }
    for (int r = threadIdx.x; r < nb; r += blockDim.x) xi[(int64_t)r * nrhs] = ys[r];
    __syncthreads();
  }
}

// x_r -= L_ri y_i for every present tile (r, i), r > i; CTA = 16 rows of one tile
constexpr int kGemvRows = 16;
__global__ void __launch_bounds__(256) gemv_fwd_kernel(Grid g, int i, double* x,
                                                       int64_t nrhs, int nrb) {
  const int r_tile = i + 1 + blockIdx.x / nrb;
  const int rb = blockIdx.x % nrb;
  TileRef T;
  if (!g.owns_row(r_tile) || !tile_ref(g, r_tile, i, T)) return;
  const int nb = g.nb;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* yi = x + (int64_t)i * nb * nrhs;
  double* xr = x + (int64_t)r_tile * nb * nrhs;
  for (int rr = warp; rr < kGemvRows; rr += 8) {
    const int r = rb * kGemvRows + rr;
    if (r >= nb) break;
    for (int64_t c = 0; c < nrhs; ++c) {
      double s = 0.0;
      for (int q = lane; q < nb; q += 32) s += T.at((int64_t)r * nb + q) * yi[(int64_t)q * nrhs + c];
      s = warp_sum(s);
      if (lane == 0) xr[(int64_t)r * nrhs + c] -= s;
    }
  }
}

// ---------------------------------------------------------- backward sweep
// x_i = L_ii^{-T} x_i, one CTA
__global__ void __launch_bounds__(512) trsv_bwd_diag_kernel(Grid g, int i, double* x,
                                                            int64_t nrhs) {
  const double* L = g.dtile(i, i);
  const int nb = g.nb;
  extern __shared__ double ys[];
  __shared__ double part[16][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  for (int64_t c = 0; c < nrhs; ++c) {
    double* xi = x + (int64_t)i * nb * nrhs + c;
    for (int r = threadIdx.x; r < nb; r += blockDim.x) ys[r] = xi[(int64_t)r * nrhs];
    __syncthreads();
    const int nblk = (nb + 31) / 32;
    for (int b = nblk - 1; b >= 0; --b) {
      const int cb = b * 32, w = min(32, nb - cb);
      const int r_lo = cb + w;
      // ys[cb + lane] -= sum_{r >= r_lo} L[r][cb + lane] ys[r]  (lanes = columns, warps = rows)
      if (r_lo < nb) {
        double s = 0.0;
        if (lane < w)
          for (int r = r_lo + warp; r < nb; r += nw) s += L[(int64_t)r * nb + cb + lane] * ys[r];
        part[warp][lane] = s;
        __syncthreads();
        if (warp == 0) {
          double t = 0.0;
          for (int q = 0; q < nw; ++q) t += part[q][lane];
          if (lane < w) ys[cb + lane] -= t;
        }
        __syncthreads();
      }
      if (warp == 0) {
        // stage column `lane` of the diagonal block (L[cb+q][cb+lane]) in registers
        double lc[32];
#pragma unroll
        for (int q = 0; q < 32; ++q)
          lc[q] = (lane < w && q < w) ? L[(int64_t)(cb + q) * nb + cb + lane] : 1.0;
        double acc = lane < w ? ys[cb + lane] : 0.0;
#pragma unroll
        for (int q = 31; q >= 0; --q) {
          if (q < w) {
            const double dq = __shfl_sync(0xffffffffu, lc[q], q);
            const double xq = __shfl_sync(0xffffffffu, acc, q) / dq;
            if (lane == q) acc = xq;
            else if (lane < q) acc -= lc[q] * xq;
          }
        }
        if (lane < w) ys[cb + lane] = acc;
      }
      __syncthreads();
    }
    for (int r = threadIdx.x; r < nb; r += blockDim.x) xi[(int64_t)r * nrhs] = ys[r];
    __syncthreads();
  }
}

// x_j -= L_ij^T x_i for every present (i, j), j < i; CTA = 32 columns of one tile
__global__ void __launch_bounds__(256) gemvt_bwd_kernel(Grid g, int i, double* x,
                                                        int64_t nrhs, int ncb) {
  const int j = blockIdx.x / ncb;
  const int cb = (blockIdx.x % ncb) * 32;
  TileRef T;
  if (!tile_ref(g, i, j, T)) return;
  const int nb = g.nb;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ double part[8][33];
  const double* xi = x + (int64_t)i * nb * nrhs;
  double* xj = x + (int64_t)j * nb * nrhs;
  const int col = cb + lane;
  for (int64_t c = 0; c < nrhs; ++c) {
    double s = 0.0;
    if (col < nb)
      for (int r = warp; r < nb; r += 8) s += T.at((int64_t)r * nb + col) * xi[(int64_t)r * nrhs + c];
    part[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && col < nb) {
      double t = 0.0;
      for (int q = 0; q < 8; ++q) t += part[q][lane];
      xj[(int64_t)col * nrhs + c] -= t;
    }
    __syncthreads();
  }
}

// --------------------------------------------------------------- dot / matvec
__global__ void __launch_bounds__(256) sumsq_partial_kernel(const double* y, int64_t m,
                                                            double* partial) {
  double s = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x)
    s += y[e] * y[e];
  __shared__ double red[8];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    partial[blockIdx.x] = t;
  }
}

// out = L v ; CTA = 16 rows of tile row i, loops over tiles j <= i
__global__ void __launch_bounds__(256) matvec_lower_kernel(Grid g, const double* v, double* out,
                                                           int nrb) {
  const int i = blockIdx.x / nrb;
  const int rb = blockIdx.x % nrb;
  const int nb = g.nb;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int rr = warp; rr < kGemvRows; rr += 8) {
    const int r = rb * kGemvRows + rr;
    if (r >= nb) break;
    double acc = 0.0;
    for (int j = 0; j <= i; ++j) {
      TileRef T;
      if (!tile_ref(g, i, j, T)) continue;
      const int qmax = (j == i) ? r + 1 : nb;
      double s = 0.0;
      for (int q = lane; q < qmax; q += 32) s += T.at((int64_t)r * nb + q) * v[(int64_t)j * nb + q];
      acc += warp_sum(s);
    }
    if (lane == 0) out[(int64_t)i * nb + r] = acc;
  }
}

}  // namespace

int mt_logdet_impl(const Grid& g, double* out, double* work, cudaStream_t st) {
  ProfScope ps(MT_K_MISC, st, 0.0, (double)g.p * g.nb * 8.0, 2);
  logdet_partial_kernel<<<g.p, 256, 0, st>>>(g, work);
  MT_LAUNCH_CHECK("logdet_partial");
  fixed_sum_kernel<<<1, 1, 0, st>>>(work, g.p, 2.0, out);
  MT_LAUNCH_CHECK("fixed_sum");
  return MT_OK;
}

int mt_solve_impl(const Grid& g, double* x, int64_t nrhs, int which, cudaStream_t st) {
  const int nb = g.nb, p = g.p;
  const size_t smem = (size_t)nb * sizeof(double);
  cudaFuncSetAttribute(trsv_fwd_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(smem > 48 * 1024 ? smem : 48 * 1024));
  cudaFuncSetAttribute(trsv_bwd_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(smem > 48 * 1024 ? smem : 48 * 1024));
  // bytes: the factor is read once per sweep
  const double fbytes = (double)g.nband() * nb * nb * 8.0 + (double)g.noff() * nb * nb * 4.0;
  const double fflops = 2.0 * (double)g.n * g.n;  // ~n^2 multiply-adds per sweep per rhs
  if (which & 1) {
    ProfScope ps(MT_K_SOLVE, st, fflops * nrhs, fbytes, 2 * p - 1);
    const int nrb = (nb + kGemvRows - 1) / kGemvRows;
    for (int i = 0; i < p; ++i) {
      trsv_fwd_diag_kernel<<<1, 512, smem, st>>>(g, i, x, nrhs);
      MT_LAUNCH_CHECK("trsv_fwd_diag");
      if (i + 1 < p) {
        gemv_fwd_kernel<<<(unsigned)((p - i - 1) * nrb), 256, 0, st>>>(g, i, x, nrhs, nrb);
        MT_LAUNCH_CHECK("gemv_fwd");
      }
    }
  }
  if (which & 2) {
    ProfScope ps(MT_K_SOLVE, st, fflops * nrhs, fbytes, 2 * p - 1);
    const int ncb = (nb + 31) / 32;
    for (int i = p - 1; i >= 0; --i) {
      trsv_bwd_diag_kernel<<<1, 512, smem, st>>>(g, i, x, nrhs);
      MT_LAUNCH_CHECK("trsv_bwd_diag");
      if (i > 0) {
        gemvt_bwd_kernel<<<(unsigned)(i * ncb), 256, 0, st>>>(g, i, x, nrhs, ncb);
        MT_LAUNCH_CHECK("gemvt_bwd");
      }
    }
  }
  return MT_OK;
}

// multi-GPU forward sweep, step i: on the owner of tile (i, i) y_i = L_ii^{-1} x_i
// (which = 1), on the ranks of tile column i x_r -= L_ri y_i for their rows r > i
// (which = 2) -- the same kernels and order as mt_solve_impl
int mt_fwd_step_impl(const Grid& g, int i, double* x, cudaStream_t st, int which) {
  const int nb = g.nb, p = g.p;
  if (((which & 1) && !g.owns(i, i)) || ((which & 2) && !g.owns_col(i))) {
    mt_set_error("rank does not own the tiles of forward-sweep step %d", i);
    return MT_E_BAD_ARG;
  }
  const size_t smem = (size_t)nb * sizeof(double);
  cudaFuncSetAttribute(trsv_fwd_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(smem > 48 * 1024 ? smem : 48 * 1024));
  ProfScope ps(MT_K_SOLVE, st, 2.0 * (double)nb * nb * (p - i), (double)nb * nb * 8.0 * (p - i), 2);
  if (which & 1) {
    trsv_fwd_diag_kernel<<<1, 512, smem, st>>>(g, i, x, 1);
    MT_LAUNCH_CHECK("trsv_fwd_diag");
  }
  if ((which & 2) && i + 1 < p) {
    const int nrb = (nb + kGemvRows - 1) / kGemvRows;
    gemv_fwd_kernel<<<(unsigned)((p - i - 1) * nrb), 256, 0, st>>>(g, i, x, 1, nrb);
    MT_LAUNCH_CHECK("gemv_fwd");
  }
  return MT_OK;
}

// per-diagonal-tile log-sums (0 for tiles another rank owns); fixed-order sum elsewhere
int mt_logdet_partials_impl(const Grid& g, double* partial, cudaStream_t st) {
  ProfScope ps(MT_K_MISC, st, 0.0, (double)g.p * g.nb * 8.0);
  logdet_partial_kernel<<<g.p, 256, 0, st>>>(g, partial);
  MT_LAUNCH_CHECK("logdet_partial");
  return MT_OK;
}

// sum of squares of m doubles with the fixed-order reduction used by mt_quad
// (work: >= 1024 doubles)
int mt_sumsq_impl(const double* x, int64_t m, double* work, double* out, cudaStream_t st) {
  const int blocks = 1024;
  ProfScope ps(MT_K_MISC, st, 2.0 * m, m * 8.0, 2);
  sumsq_partial_kernel<<<blocks, 256, 0, st>>>(x, m, work);
  MT_LAUNCH_CHECK("sumsq_partial");
  fixed_sum_kernel<<<1, 1, 0, st>>>(work, blocks, 1.0, out);
  MT_LAUNCH_CHECK("fixed_sum");
  return MT_OK;
}

// work: n_pad doubles (y) + 1024 partials
int mt_quad_impl(const Grid& g, const double* z, double* work, double* out, cudaStream_t st) {
  const int64_t npad = (int64_t)g.p * g.nb;
  if (mt_cuda_check(cudaMemcpyAsync(work, z, npad * sizeof(double), cudaMemcpyDeviceToDevice, st),
                    "quad copy"))
    return MT_E_CUDA;
  int rc = mt_solve_impl(g, work, 1, 1, st);
  if (rc) return rc;
  double* partial = work + npad;
  const int blocks = 1024;
  ProfScope ps(MT_K_MISC, st, 2.0 * npad, npad * 8.0, 2);
  sumsq_partial_kernel<<<blocks, 256, 0, st>>>(work, npad, partial);
  MT_LAUNCH_CHECK("sumsq_partial");
  fixed_sum_kernel<<<1, 1, 0, st>>>(partial, blocks, 1.0, out);
  MT_LAUNCH_CHECK("fixed_sum");
  return MT_OK;
}

int mt_matvec_lower_impl(const Grid& g, const double* v, double* out, cudaStream_t st) {
  const int nrb = (g.nb + kGemvRows - 1) / kGemvRows;
  ProfScope ps(MT_K_SOLVE, st, (double)g.n * g.n, (double)g.nband() * g.nb * g.nb * 8.0);
  matvec_lower_kernel<<<(unsigned)(g.p * nrb), 256, 0, st>>>(g, v, out, nrb);
  MT_LAUNCH_CHECK("matvec_lower");
  return MT_OK;
}
