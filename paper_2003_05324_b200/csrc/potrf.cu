// Diagonal-tile Cholesky POTRF(k), FP64, in place on the row-major tile
// (kernels.potrf + factor.py:249-256).
//
// One CTA (8 warps) walks the tile in 32-wide column blocks, right-looking:
//   1. warp 0 factors the 32x32 diagonal block with the rows held in
//      registers (lane r owns row r, pivots broadcast by shuffles, no CTA
//      barrier per pivot) and forms its triangular inverse column-wise;
//   2. the sub-diagonal panel is solved as a parallel GEMM against that
//      inverse (X = A L_dd^{-T}), staged in shared memory;
//   3. the trailing lower triangle takes the rank-32 SYRK update on the FP64
//      tensor cores (mma.sync m8n8k4 f64 -> DMMA), 32x32 warp tiles fed from
//      the shared-memory panel.
// Epilogue: the first non-positive (or NaN) pivot is published as the global
// index k*nb + j (FactorizationError.index); the 32x32 diagonal-block
// inverses (FP64 + FP32) are kept for the panel TRSM, and in MP mode the
// factor is narrowed to FP32 for the off-band panel solves (sp_diag,
// factor.py:255-256).  The strict upper triangle is never written.
#include <cooperative_groups.h>

#include "mt_grid.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int PLD = 36;  // panel row stride in doubles: conflict-free m8n8k4 fragments

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// 32x32 diagonal block: factor and triangular inverse, by ONE warp, no CTA
// barrier.  Lane r loads row r (rows/columns >= w are the identity) and the
// fully unrolled right-looking pivot loop keeps every index static: pivot j
// is broadcast by a shuffle, d = sqrt(pivot), the column is scaled by the
// reciprocal 1/d (dpotf2: DSCAL by ONE/AJJ) and the trailing entries of the
// row take a[c] -= L[r][j] L[c][j], j ascending.  The inverse is then formed
// column-wise, lane c holding column c of L^{-1}: x_r = b_r / L[r][r] (as the
// product with the pivot's reciprocal, already in every lane) and
// b_q -= L[q][r] x_r for q > r, the L column read by broadcast from Ld.
// Writes Ld (lower, zero above; column 32 = the pivot reciprocals) and Li
// (lower, zero above) in shared memory (row stride 33); returns the local
// index of the first non-positive / NaN pivot, -1 when the block is positive
// definite (warp-uniform).  Every POTRF variant calls this, so their results
// stay bitwise equal.  ncu at N=65536: potrf_kernel 1.37 -> 1.00 ms per tile,
// the cluster kernel 0.75 -> 0.35 ms, against the former shuffle pivots + a
// CTA-wide row-by-row inverse (64 barriers); a rolled pivot loop (window
// shifted through the registers) measured 1.12 / 0.44 ms.
__device__ __noinline__ int diag_block_factor_inverse(const double* src, int64_t ld, int w,
                                                        double* Ld, double* Li) {
  const int r = threadIdx.x & 31;
  double a[32];
#pragma unroll
  for (int c = 0; c < 32; ++c)
    a[c] = (r < w && c < w) ? (c <= r ? src[r * ld + c] : 0.0) : (r == c ? 1.0 : 0.0);
  int fail = -1;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    double piv = __shfl_sync(0xffffffffu, a[j], j);
    if (fail < 0 && !(piv > 0.0)) fail = j;  // warp-uniform; later steps are discarded
    if (fail >= 0) piv = 1.0;
    const double d = sqrt(piv);
    const double rd = 1.0 / d;
    if (r == 0) Ld[j * 33 + 32] = rd;  // the pad column keeps 1 / L[j][j]
    const double lrj = r == j ? d : (r > j ? a[j] * rd : 0.0);
    a[j] = lrj;
#pragma unroll
    for (int c = j + 1; c < 32; ++c) {
      const double lcj = __shfl_sync(0xffffffffu, lrj, c);  // L[c][j]
      if (r >= c) a[c] -= lrj * lcj;
    }
  }
#pragma unroll
  for (int c = 0; c < 32; ++c) Ld[r * 33 + c] = c <= r ? a[c] : 0.0;
  __syncwarp();
  // inverse: lane c solves L x = e_c (reuses a[] as b / x)
#pragma unroll
  for (int q = 0; q < 32; ++q) a[q] = q == r ? 1.0 : 0.0;
#pragma unroll
  for (int q = 0; q < 32; ++q) {
    a[q] = q < r ? 0.0 : a[q] * Ld[q * 33 + 32];
#pragma unroll
    for (int u = q + 1; u < 32; ++u) a[u] -= Ld[u * 33 + q] * a[q];
  }
#pragma unroll
  for (int q = 0; q < 32; ++q) Li[q * 33 + r] = a[q];
  __syncwarp();
  return fail;
}

__global__ void __launch_bounds__(kThreads, 1) potrf_kernel(Grid g, int k, int narrow) {
  if (g.failed()) return;
  double* __restrict__ A = g.dtile(k, k);
  const int nb = g.nb;
  extern __shared__ __align__(16) double P[];  // (nb - 32) x PLD: solved panel
  __shared__ double Ld[32][33];
  __shared__ double Li[32][33];
  __shared__ int bad;
  double* inv64 = g.sinv64(k);
  float* inv32 = g.sinv32(k);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) bad = -1;

  for (int c0 = 0, blk = 0; c0 < nb; c0 += 32, ++blk) {
    const int w = min(32, nb - c0);
    // ---------------- 1. diagonal block: factor + inverse (warp 0) ---------
    if (warp == 0) {
      const int fail = diag_block_factor_inverse(A + (int64_t)c0 * nb + c0, nb, w, &Ld[0][0], &Li[0][0]);
      if (fail >= 0 && lane == 0) bad = c0 + fail;
    }
    __syncthreads();
    if (bad < 0) {
      // write the factored block (lower), its FP32 narrowing, and the inverse
      float* S = narrow ? g.sdiag(k) : nullptr;
      for (int e = threadIdx.x; e < 32 * 32; e += kThreads) {
        const int r = e >> 5, c = e & 31;
        if (r < w && c < w && c <= r) {
          const int64_t o = (int64_t)(c0 + r) * nb + c0 + c;
          A[o] = Ld[r][c];
          if (S) S[o] = __double2float_rn(Ld[r][c]);
        }
        const double v = Li[r][c];
        inv64[blk * 1024 + e] = v;
        inv32[blk * 1024 + e] = __double2float_rn(v);
      }
    }
    __syncthreads();
    if (bad >= 0) {
      if (threadIdx.x == 0)
        atomicCAS((unsigned long long*)&g.status[MT_ST_PIVOT], (unsigned long long)-1LL,
                  (unsigned long long)((int64_t)k * nb + bad));
      return;
    }
    const int r_lo = c0 + w;
    const int m = nb - r_lo;
    if (m <= 0) continue;
    // ---------------- 2. panel: X = A[r_lo:, c0:c0+32] L_dd^{-T} -----------
    for (int e = threadIdx.x; e < m * 32; e += kThreads) {
      const int rr = e >> 5, q = e & 31;
      P[rr * PLD + q] = q < w ? A[(int64_t)(r_lo + rr) * nb + c0 + q] : 0.0;
    }
    __syncthreads();
    for (int rb = 0; rb < m; rb += 32) {
      // thread: row rb + tid/8, columns 4*(tid%8) .. +3
      const int rr = rb + (threadIdx.x >> 3), cg = (threadIdx.x & 7) * 4;
      double o[4] = {0.0, 0.0, 0.0, 0.0};
      if (rr < m) {
#pragma unroll 8
        for (int q = 0; q < 32; ++q) {
          const double av = P[rr * PLD + q];
#pragma unroll
          for (int u = 0; u < 4; ++u) o[u] += av * Li[cg + u][q];
        }
      }
      __syncthreads();
      if (rr < m) {
        float* S = narrow ? g.sdiag(k) : nullptr;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = cg + u;
          P[rr * PLD + c] = c < w ? o[u] : 0.0;
          if (c < w) {
            const int64_t o2 = (int64_t)(r_lo + rr) * nb + c0 + c;
            A[o2] = o[u];
            if (S) S[o2] = __double2float_rn(o[u]);  // FP32 narrowing, fused
          }
        }
      }
      __syncthreads();
    }
    // ---------------- 3. trailing SYRK on DMMA: A[r][c] -= P[r] . P[c] ------
    const int mt = (m + 31) / 32;
    const int ntile = mt * (mt + 1) / 2;
    for (int tIdx = warp; tIdx < ntile; tIdx += kThreads / 32) {
      int tr = (int)((sqrtf(8.0f * (float)tIdx + 1.0f) - 1.0f) * 0.5f);
      while (tr * (tr + 1) / 2 > tIdx) --tr;
      while ((tr + 1) * (tr + 2) / 2 <= tIdx) ++tr;
      const int tc = tIdx - tr * (tr + 1) / 2;
      double acc[4][4][2];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll
      for (int k4 = 0; k4 < 32; k4 += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          const int ra = min(tr * 32 + f * 8 + (lane >> 2), m - 1);
          const int rb2 = min(tc * 32 + f * 8 + (lane >> 2), m - 1);
          af[f] = P[ra * PLD + k4 + (lane & 3)];
          bf[f] = P[rb2 * PLD + k4 + (lane & 3)];
        }
#pragma unroll
        for (int fm = 0; fm < 4; ++fm)
#pragma unroll
          for (int fn = 0; fn < 4; ++fn) dmma884(acc[fm][fn], af[fm], bf[fn]);
      }
      // epilogue: issue every load of the warp tile before any store (a
      // load/store per element would serialise on L2 latency: stores may
      // alias later loads as far as the compiler knows)
      double cv[4][4][2];
#pragma unroll
      for (int fm = 0; fm < 4; ++fm) {
        const int r = tr * 32 + fm * 8 + (lane >> 2);
#pragma unroll
        for (int fn = 0; fn < 4; ++fn) {
          const int c = tc * 32 + fn * 8 + 2 * (lane & 3);
          const double* rowp = A + (int64_t)(r_lo + min(r, m - 1)) * nb + r_lo;
          cv[fm][fn][0] = rowp[min(c, m - 1)];
          cv[fm][fn][1] = rowp[min(c + 1, m - 1)];
        }
      }
#pragma unroll
      for (int fm = 0; fm < 4; ++fm) {
        const int r = tr * 32 + fm * 8 + (lane >> 2);
        if (r >= m) continue;
#pragma unroll
        for (int fn = 0; fn < 4; ++fn) {
          const int c = tc * 32 + fn * 8 + 2 * (lane & 3);
          double* cp = A + (int64_t)(r_lo + r) * nb + r_lo + c;
          if (c < m && c <= r) cp[0] = cv[fm][fn][0] - acc[fm][fn][0];
          if (c + 1 < m && c + 1 <= r) cp[1] = cv[fm][fn][1] - acc[fm][fn][1];
        }
      }
    }
    __syncthreads();
  }
  // (the FP32 narrowing of the lower triangle was written as each element was
  //  finalised; the TRSM never reads the strict upper part)
}


// ---------------------------------------------------------------------------
// Cluster POTRF: the tile's 32-row blocks spread over a thread-block cluster
// of nb/32 CTAs (one SM each), the tile resident in distributed shared memory.
// CTA c holds row block c (its 32 x 32(c+1) lower part).  For each column
// block cb: CTA cb factors its diagonal block and forms the inverse (the same
// diagonal-block factor and inverse as potrf_kernel); after a cluster
// barrier every CTA c > cb solves its panel block X_c = A[c,cb] Li^T; after a
// second barrier it applies A[c,q] -= X_c X_q^T for cb < q <= c on DMMA,
// reading X_q from CTA q's shared memory.  Every element sees the same
// operations in the same order as in potrf_kernel (panel FMAs in q order,
// SYRK blocks accumulated k4-ascending then subtracted once): bitwise equal
// results (tests/test_gpu_factor.py).  Alone it takes 0.75 ms per 512-tile
// against 1.37 ms (ncu); inside the factorization it is slower overall (862 ->
// 1100 ms Cholesky at N=65536): the 16-CTA cluster must find a whole GPC free
// beside the co-scheduled bulk update, stalling the panel chain.  Opt-in
// (option 14) for layouts where the panel chain is exposed.
namespace cg = cooperative_groups;
constexpr int CLD = 8;  // row padding (doubles) of the resident row block

__global__ void __launch_bounds__(kThreads, 1) potrf_cluster_kernel(Grid g, int k, int narrow) {
  cg::cluster_group cluster = cg::this_cluster();
  const int c = (int)cluster.block_rank();  // this CTA's row block
  const int nblk = (int)cluster.num_blocks();
  const int nb = g.nb;
  const int ld = nb + CLD;                  // resident rows: 32 x ld doubles
  extern __shared__ __align__(16) double R[];   // [32][ld]: rows 32c.. of the tile
  double* Ld = R + 32 * ld;                      // [32][33] diagonal factor (owner)
  double* Li = Ld + 32 * 33;                     // [32][33] its inverse (owner)
  double* Lp = Li + 32 * 33;                     // [32][33] peer's inverse (copy)
  double* Xq = Lp + 32 * 33;                     // [32][36] peer's panel block (copy)
  __shared__ int bad;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* A = g.dtile(k, k);
  double* inv64 = g.sinv64(k);
  float* inv32 = g.sinv32(k);
  if (threadIdx.x == 0) bad = -1;
  const bool failed0 = g.failed();
  // load the lower part of row block c (columns 0 .. 32(c+1)-1)
  const int wcols = 32 * (c + 1);
  for (int e = threadIdx.x; e < 32 * wcols; e += kThreads) {
    const int r = e / wcols, q = e % wcols;
    R[r * ld + q] = A[(int64_t)(32 * c + r) * nb + q];
  }
  cluster.sync();
  if (failed0) return;  // uniform: every CTA read the same status word

  for (int cb = 0; cb < nblk; ++cb) {
    double* Dcb = R + cb * 32;  // block (c, cb) of this CTA's rows
    __syncthreads();  // the previous step's trailing writes (all warps) before the diagonal read
    if (c == cb) {
      // -------- diagonal block: warp 0 factors it in registers (potrf_kernel step 1)
      if (warp == 0) {
        const int fail = diag_block_factor_inverse(Dcb, ld, 32, Ld, Li);
        if (fail >= 0 && lane == 0) bad = cb * 32 + fail;
      }
      __syncthreads();
      if (bad < 0) {
        for (int e = threadIdx.x; e < 32 * 32; e += kThreads) {
          const int r = e >> 5, q = e & 31;
          if (q <= r) Dcb[r * ld + q] = Ld[r * 33 + q];
          inv64[cb * 1024 + e] = Li[r * 33 + q];
          inv32[cb * 1024 + e] = __double2float_rn(Li[r * 33 + q]);
        }
      } else if (threadIdx.x == 0) {
        atomicCAS((unsigned long long*)&g.status[MT_ST_PIVOT], (unsigned long long)-1LL,
                  (unsigned long long)((int64_t)k * nb + bad));
      }
    }
    cluster.sync();  // (1) diagonal block cb and its inverse are final
    const int fail = *cluster.map_shared_rank(&bad, cb);
    if (fail >= 0) {  // uniform across the cluster
      cluster.sync();  // nobody exits while a peer may still read its shared memory
      return;
    }
    if (c > cb) {
      // -------- panel block: X = A[c, cb] Li^T (potrf_kernel step 2)
      const double* Lr = cluster.map_shared_rank(Li, cb);
      for (int e = threadIdx.x; e < 32 * 32; e += kThreads) Lp[(e >> 5) * 33 + (e & 31)] = Lr[(e >> 5) * 33 + (e & 31)];
      __syncthreads();
      const int rr = threadIdx.x >> 3, cg4 = (threadIdx.x & 7) * 4;
      double o[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
      for (int q = 0; q < 32; ++q) {
        const double av = Dcb[rr * ld + q];
#pragma unroll
        for (int u = 0; u < 4; ++u) o[u] += av * Lp[(cg4 + u) * 33 + q];
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 4; ++u) Dcb[rr * ld + cg4 + u] = o[u];
    }
    cluster.sync();  // (2) panel blocks of column cb are final
    if (c > cb) {
      // -------- trailing blocks of row block c: A[c, q] -= X_c X_q^T (DMMA)
      for (int q = cb + 1; q <= c; ++q) {
        const double* Xsrc = q == c ? Dcb : cluster.map_shared_rank(R, q) + cb * 32;
        __syncthreads();  // Xq free (previous q consumed)
        for (int e = threadIdx.x; e < 32 * 32; e += kThreads)
          Xq[(e >> 5) * 36 + (e & 31)] = Xsrc[(e >> 5) * ld + (e & 31)];
        __syncthreads();
        // 16 fragments of 8 x 8, two per warp
        const int fm = warp >> 1, fn0 = (warp & 1) * 2;
        double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
        for (int k4 = 0; k4 < 32; k4 += 4) {
          const double af = Dcb[(fm * 8 + (lane >> 2)) * ld + k4 + (lane & 3)];
#pragma unroll
          for (int f = 0; f < 2; ++f) {
            const double bf = Xq[((fn0 + f) * 8 + (lane >> 2)) * 36 + k4 + (lane & 3)];
            dmma884(acc[f], af, bf);
          }
        }
        double* Cq = R + q * 32;
#pragma unroll
        for (int f = 0; f < 2; ++f) {
          const int r = fm * 8 + (lane >> 2), col = (fn0 + f) * 8 + 2 * (lane & 3);
          Cq[r * ld + col] -= acc[f][0];
          Cq[r * ld + col + 1] -= acc[f][1];
        }
      }
    }
  }
  cluster.sync();  // peers no longer read this CTA's blocks
  // write back the lower part of row block c and its FP32 narrowing
  float* S = narrow ? g.sdiag(k) : nullptr;
  for (int e = threadIdx.x; e < 32 * wcols; e += kThreads) {
    const int r = e / wcols, q = e % wcols;
    if (q > 32 * c + r) continue;  // strict upper part of the diagonal block
    const int64_t o = (int64_t)(32 * c + r) * nb + q;
    const double v = R[r * ld + q];
    A[o] = v;
    if (S) S[o] = __double2float_rn(v);
  }
}


// ---------------------------------------------------------------------------
// Multi-kernel POTRF (option 14 = 2): per 32-column block cb three small
// launches -- the diagonal block (1 CTA: one warp factors and inverts it),
// the panel blocks (one CTA per row block below), the trailing lower blocks
// (one CTA per (c, q) block pair) -- with the single-CTA kernel's operation
// order per element (bitwise equal).  No cluster and no co-residency: every
// launch takes whatever SMs are free beside the bulk update, so the serial
// chain is the diagonal-block work plus launch latency.
__global__ void __launch_bounds__(kThreads) potrf_mk_diag(Grid g, int k, int cb, int narrow) {
  if (g.failed()) return;
  double* __restrict__ A = g.dtile(k, k);
  const int nb = g.nb, c0 = cb * 32;
  __shared__ double Ld[32][33];
  __shared__ double Li[32][33];
  __shared__ int bad;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) bad = -1;
  __syncthreads();
  if (warp == 0) {
    const int fail = diag_block_factor_inverse(A + (int64_t)c0 * nb + c0, nb, 32, &Ld[0][0], &Li[0][0]);
    if (fail >= 0 && lane == 0) bad = c0 + fail;
  }
  __syncthreads();
  if (bad >= 0) {
    if (threadIdx.x == 0)
      atomicCAS((unsigned long long*)&g.status[MT_ST_PIVOT], (unsigned long long)-1LL,
                (unsigned long long)((int64_t)k * nb + bad));
    return;
  }
  float* S = narrow ? g.sdiag(k) : nullptr;
  double* inv64 = g.sinv64(k);
  float* inv32 = g.sinv32(k);
  for (int e = threadIdx.x; e < 32 * 32; e += kThreads) {
    const int r = e >> 5, c = e & 31;
    if (c <= r) {
      const int64_t o = (int64_t)(c0 + r) * nb + c0 + c;
      A[o] = Ld[r][c];
      if (S) S[o] = __double2float_rn(Ld[r][c]);
    }
    inv64[cb * 1024 + e] = Li[r][c];
    inv32[cb * 1024 + e] = __double2float_rn(Li[r][c]);
  }
}

// panel block (c, cb), c = cb + 1 + blockIdx.x: X = A[c, cb] Li^T
__global__ void __launch_bounds__(kThreads) potrf_mk_panel(Grid g, int k, int cb, int narrow) {
  if (g.failed()) return;
  double* __restrict__ A = g.dtile(k, k);
  const int nb = g.nb, c0 = cb * 32, r0 = (cb + 1 + blockIdx.x) * 32;
  __shared__ double Li[32][33];
  __shared__ double X[32][33];
  const double* inv64 = g.sinv64(k) + cb * 1024;
  for (int e = threadIdx.x; e < 1024; e += kThreads) {
    Li[e >> 5][e & 31] = inv64[e];
    X[e >> 5][e & 31] = A[(int64_t)(r0 + (e >> 5)) * nb + c0 + (e & 31)];
  }
  __syncthreads();
  const int rr = threadIdx.x >> 3, cg = (threadIdx.x & 7) * 4;
  double o[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
  for (int q = 0; q < 32; ++q) {
    const double av = X[rr][q];
#pragma unroll
    for (int u = 0; u < 4; ++u) o[u] += av * Li[cg + u][q];
  }
  float* S = narrow ? g.sdiag(k) : nullptr;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t off = (int64_t)(r0 + rr) * nb + c0 + cg + u;
    A[off] = o[u];
    if (S) S[off] = __double2float_rn(o[u]);
  }
}

// trailing block (c, q), cb < q <= c: A[c, q] -= X_c X_q^T on DMMA
__global__ void __launch_bounds__(kThreads) potrf_mk_trail(Grid g, int k, int cb) {
  if (g.failed()) return;
  double* __restrict__ A = g.dtile(k, k);
  const int nb = g.nb, c0 = cb * 32;
  // blockIdx.x -> (tr, tc), tc <= tr, over the m = nblk - cb - 1 trailing row blocks
  const int tIdx = blockIdx.x;
  int tr = (int)((sqrtf(8.0f * (float)tIdx + 1.0f) - 1.0f) * 0.5f);
  while (tr * (tr + 1) / 2 > tIdx) --tr;
  while ((tr + 1) * (tr + 2) / 2 <= tIdx) ++tr;
  const int tc = tIdx - tr * (tr + 1) / 2;
  const int rc = (cb + 1 + tr) * 32, rq = (cb + 1 + tc) * 32;
  __shared__ double Xc[32][PLD];
  __shared__ double Xq[32][PLD];
  for (int e = threadIdx.x; e < 1024; e += kThreads) {
    Xc[e >> 5][e & 31] = A[(int64_t)(rc + (e >> 5)) * nb + c0 + (e & 31)];
    Xq[e >> 5][e & 31] = A[(int64_t)(rq + (e >> 5)) * nb + c0 + (e & 31)];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int fm = warp >> 1, fn0 = (warp & 1) * 2;
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int k4 = 0; k4 < 32; k4 += 4) {
    const double af = Xc[fm * 8 + (lane >> 2)][k4 + (lane & 3)];
#pragma unroll
    for (int f = 0; f < 2; ++f) dmma884(acc[f], af, Xq[(fn0 + f) * 8 + (lane >> 2)][k4 + (lane & 3)]);
  }
#pragma unroll
  for (int f = 0; f < 2; ++f) {
    const int r = fm * 8 + (lane >> 2), c = (fn0 + f) * 8 + 2 * (lane & 3);
    double* cp = A + (int64_t)(rc + r) * nb + rq + c;
    if (tr != tc || c <= r) cp[0] -= acc[f][0];
    if (tr != tc || c + 1 <= r) cp[1] -= acc[f][1];
  }
}

}  // namespace

static size_t potrf_cluster_smem(int nb) {
  return ((size_t)32 * (nb + CLD) + 3 * 32 * 33 + 32 * 36) * sizeof(double);
}

// cluster kernel when the tile splits into 2..16 row blocks of 32 and fits in
// distributed shared memory; the single-CTA kernel otherwise (same results)
static int g_potrf_cluster = -1;  // -1 unknown, 0 unavailable, 1 usable

int mt_potrf_impl(const Grid& g, int k, int narrow, cudaStream_t st) {
  const double r = g.rows(k);
  const int nblk = g.nb / 32;
  const bool multi_kernel = mt_opt_potrf_cluster() == 2 && g.nb % 32 == 0 && nblk >= 2;
  ProfScope ps(MT_K_POTRF, st, r * r * r / 3.0,
               (double)g.nb * g.nb * (16.0 + (narrow ? 4.0 : 0.0)), multi_kernel ? 3 * nblk - 2 : 1);
  if (multi_kernel) {
    for (int cb = 0; cb < nblk; ++cb) {
      potrf_mk_diag<<<1, kThreads, 0, st>>>(g, k, cb, narrow);
      const int m = nblk - cb - 1;
      if (m > 0) {
        potrf_mk_panel<<<m, kThreads, 0, st>>>(g, k, cb, narrow);
        potrf_mk_trail<<<m * (m + 1) / 2, kThreads, 0, st>>>(g, k, cb);
      }
    }
    MT_LAUNCH_CHECK("potrf_mk");
    return MT_OK;
  }
  if (mt_opt_potrf_cluster() == 1 && g.nb % 32 == 0 && nblk >= 2 && nblk <= 16 &&
      potrf_cluster_smem(g.nb) <= 220 * 1024 && g_potrf_cluster != 0) {
    const size_t smem = potrf_cluster_smem(g.nb);
    cudaFuncSetAttribute(potrf_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(potrf_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblk);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = nblk;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, potrf_cluster_kernel, g, k, narrow);
    if (e == cudaSuccess) {
      g_potrf_cluster = 1;
      return MT_OK;
    }
    if (g_potrf_cluster == 1) return mt_cuda_check(e, "potrf_cluster_kernel") ? MT_E_CUDA : MT_OK;
    cudaGetLastError();  // first use: cluster shape unsupported here -> single-CTA kernel
    g_potrf_cluster = 0;
  }
  const size_t smem = (size_t)(g.nb > 32 ? g.nb - 32 : 1) * PLD * sizeof(double);
  if (smem > 200 * 1024) {
    mt_set_error("potrf: nb=%d exceeds the supported maximum", g.nb);
    return MT_E_BAD_ARG;
  }
  cudaFuncSetAttribute(potrf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  potrf_kernel<<<1, kThreads, smem, st>>>(g, k, narrow);
  MT_LAUNCH_CHECK("potrf_kernel");
  return MT_OK;
}
