// Matern covariance tile generation (subsystem 1 of the north star).
//
// One fused pass per pool: distance (Euclidean hypot or haversine, computed
// on the fly from an N x 2 FP64 location array -- the reference instead
// caches an O(N^2) FP64 distance dict, tilestore.py:225-237), Matern value
// (closed forms at nu = 1/2, 3/2, else Temme series / Steed CF2 + upward
// recurrence, covmath.py:103-212,261-283), then a 16-byte vector store:
// FP64 for band tiles, cvt.rn.f32.f64 for off-band tiles (tile_to_sp,
// tilestore.py:103-116, including its overflow check).  Padding rows/columns
// of the last tile get identity/zero.
//
// Built with -fmad=false so the FP64 arithmetic rounds like numpy's (no
// contraction); remaining differences come from libdevice vs libm
// transcendentals (<= 2 ulp).
#include <math.h>

#include "mt_grid.cuh"

namespace {

constexpr double kEps = 2.2e-16;      // covmath.py:100
constexpr int kSeriesMax = 80;        // covmath.py:98
constexpr int kCfMax = 2000;          // covmath.py:99
constexpr double kDeg2Rad = 3.141592653589793 / 180.0;

__device__ __forceinline__ double dist(const double2 a, const double2 b, int metric,
                                       double radius) {
  if (metric == MT_METRIC_EUCLIDEAN) return hypot(a.x - b.x, a.y - b.y);
  // haversine with clipping (covmath.py:349-358); a = row point, b = column point
  double pa = a.y * kDeg2Rad, pb = b.y * kDeg2Rad;
  double dphi = pb - pa;
  double dlam = b.x * kDeg2Rad - a.x * kDeg2Rad;
  double s1 = sin(dphi / 2.0), s2 = sin(dlam / 2.0);
  double hav = s1 * s1 + cos(pa) * cos(pb) * (s2 * s2);
  hav = fmin(1.0, fmax(0.0, hav));
  return 2.0 * radius * asin(sqrt(hav));
}

// K_mu, K_{mu+1} for x <= 2 (Temme series, covmath.py:103-135)
__device__ __forceinline__ void k_series(double x, const mt_matern& th, double& k0,
                                         double& k1) {
  const double mu = th.mu;
  double lg = log(2.0 / x);
  double e = mu * lg;
  double shc = (e == 0.0) ? 1.0 : sinh(e) / e;
  double f = th.fact * (th.gam1 * cosh(e) + th.gam2 * lg * shc);
  double pp = 0.5 * exp(e) / th.rp;
  double qq = 0.5 * exp(-e) / th.rm;
  double c = 1.0, s0 = f, s1 = pp;
  const double hx2 = 0.25 * x * x;
  const double mu2 = mu * mu;
  for (int k = 1; k <= kSeriesMax; ++k) {
    double dk = (double)k;
    f = (dk * f + pp + qq) / ((double)(k * k) - mu2);
    c = c * hx2 / dk;
    pp = pp / (dk - mu);
    qq = qq / (dk + mu);
    double d0 = c * f;
    s0 = s0 + d0;
    s1 = s1 + c * (pp - dk * f);
    if (!(fabs(d0) > kEps * fabs(s0))) break;
  }
  k0 = s0;
  k1 = s1 * (2.0 / x);
}

// K_mu, K_{mu+1} for x > 2 (Steed's CF2, covmath.py:146-183)
__device__ __forceinline__ void k_cf2(double x, const mt_matern& th, double& k0, double& k1) {
  const double mu = th.mu;
  const double a1 = 0.25 - mu * mu;
  double b = 2.0 * (1.0 + x);
  double d = 1.0 / b;
  double h = d, dh = d;
  double q1 = 0.0, q2 = 1.0, q = a1, c = a1;
  double a = -a1;
  double s = 1.0 + q * dh;
  for (int i = 2; i <= kCfMax; ++i) {
    a -= 2.0 * (double)(i - 1);
    c = -a * c / (double)i;
    double qn = (q1 - b * q2) / a;
    q1 = q2;
    q2 = qn;
    q = q + c * qn;
    b = b + 2.0;
    d = 1.0 / (b + a * d);
    dh = (b * d - 1.0) * dh;
    h = h + dh;
    double ds = q * dh;
    s = s + ds;
    if (!(fabs(ds) > kEps * fabs(s))) break;
  }
  h = a1 * h;
  k0 = sqrt(3.141592653589793 / (2.0 * x)) * exp(-x) / s;
  k1 = k0 * (mu + x + 0.5 - h) / x;
}

}  // namespace

// Matern value at distance r (covmath.py:261-283); r >= 0
__device__ double mt_matern_value(double r, const mt_matern& th) {
  double z = r / th.spatial_range;
  if (th.kind == 0) return th.variance * exp(-z);
  if (th.kind == 1) return th.variance * (1.0 + z) * exp(-z);
  if (!(z > 0.0)) return th.variance;
  double k0, k1;
  if (z <= 2.0) k_series(z, th, k0, k1);
  else k_cf2(z, th, k0, k1);
  for (int j = 0; j < th.nl; ++j) {
    double kn = k0 + (2.0 * ((th.mu + (double)j) + 1.0) / z) * k1;  // (mu + j) + 1 as in Python
    k0 = k1;
    k1 = kn;
  }
  return th.scale * pow(z, th.smoothness) * k0;
}

namespace {

template <typename T>
struct Vec;
template <>
struct Vec<double> { static constexpr int W = 2; };
template <>
struct Vec<float> { static constexpr int W = 4; };

// blockIdx.x = (slot - slot0) * nrb + row block; each CTA writes kRows rows
constexpr int kRows = 8;

template <typename T>
__global__ void __launch_bounds__(256) gen_kernel(Grid g, const double2* __restrict__ locs,
                                                  int metric, double radius, mt_matern th,
                                                  int64_t slot0, int nrb) {
  const int64_t slot = slot0 + blockIdx.x / nrb;
  const int rb = blockIdx.x % nrb;
  int i, j;
  T* tile;
  if constexpr (sizeof(T) == 8) {
    g.band_slot_ij(slot, i, j);
    tile = (T*)g.dtile(i, j);
  } else {
    g.off_slot_ij(slot, i, j);
    tile = (T*)g.stile(i, j);
  }
  const int nb = g.nb;
  const int64_t n = g.n;
  const int r0 = rb * kRows;
  const int rcount = min(kRows, nb - r0);
  constexpr int W = Vec<T>::W;
  const bool vec = (nb % W) == 0;
  const int w = vec ? W : 1;
  const int nvc = nb / w;
  int local_overflow = 0;
  for (int e = threadIdx.x; e < rcount * nvc; e += blockDim.x) {
    const int r = r0 + e / nvc;
    const int c0 = (e % nvc) * w;
    const int64_t gr = (int64_t)i * nb + r;
    T out[W];
    double2 pr = make_double2(0.0, 0.0);
    if (gr < n) pr = locs[gr];
    auto elem = [&](int q) -> T {
      const int64_t gc = (int64_t)j * nb + c0 + q;
      double v;
      if (gr >= n || gc >= n) {
        v = (gr == gc) ? 1.0 : 0.0;
      } else {
        v = mt_matern_value(dist(pr, locs[gc], metric, radius), th);
      }
      if constexpr (sizeof(T) == 4) {
        float f = __double2float_rn(v);
        if (isfinite(v) && !isfinite(f)) ++local_overflow;
        return f;
      } else {
        return v;
      }
    };
    if (vec && th.kind == 0 && gr < n && (int64_t)j * nb + c0 + W <= n) {
      // nu = 1/2 interior: W independent inline FP64 chains (hypot, divide, exp;
      // same operations and order as mt_matern_value) that the compiler can
      // interleave -- generation is latency-bound on these chains
      double v[W];
#pragma unroll
      for (int q = 0; q < W; ++q) {
        const double2 pc = locs[(int64_t)j * nb + c0 + q];
        v[q] = th.variance * exp(-(dist(pr, pc, metric, radius) / th.spatial_range));
      }
#pragma unroll
      for (int q = 0; q < W; ++q) {
        if constexpr (sizeof(T) == 4) {
          const float f = __double2float_rn(v[q]);
          if (isfinite(v[q]) && !isfinite(f)) ++local_overflow;
          out[q] = f;
        } else {
          out[q] = v[q];
        }
      }
    } else if (vec) {
#pragma unroll
      for (int q = 0; q < W; ++q) out[q] = elem(q);
    } else {
      out[0] = elem(0);
    }
    T* dst = tile + (int64_t)r * nb + c0;
    if (vec) {
      if constexpr (sizeof(T) == 8) {
        *(double2*)dst = make_double2(out[0], out[1]);
      } else {
        *(float4*)dst = make_float4(out[0], out[1], out[2], out[3]);
      }
    } else {
      dst[0] = out[0];
    }
  }
  if constexpr (sizeof(T) == 4) {
    if (local_overflow) atomicAdd((unsigned long long*)&g.status[MT_ST_OVERFLOW],
                                  (unsigned long long)local_overflow);
  }
}

// zero-distance pairs a < b (duplicate locations): one CTA per row a (grid-stride)
__global__ void dup_kernel(const double2* __restrict__ locs, int64_t n, int metric,
                           double radius, int64_t* status) {
  unsigned long long cnt = 0;
  for (int64_t a = blockIdx.x; a < n; a += gridDim.x) {
    const double2 pa = locs[a];
    for (int64_t b = threadIdx.x; b < a; b += blockDim.x)
      if (dist(pa, locs[b], metric, radius) == 0.0) ++cnt;
  }
  if (cnt) atomicAdd((unsigned long long*)&status[MT_ST_DUP], cnt);
}

__global__ void matern_array_kernel(const double* __restrict__ r, int64_t m, mt_matern th,
                                    double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = mt_matern_value(r[e], th);
}

// Kriging cross-covariance product (predict.krige, predict.py:37-49):
//   out[a] = sum_b C(d(test_a, train_b)) w[b]
// without materialising the m x n cross-covariance.  blockIdx.x covers kTP
// test points, blockIdx.y one chunk of kChunk training points; each thread
// reuses a loaded training point for all kTP test points.  Partials are
// reduced in a fixed order (shuffle tree, then warps in order, then chunks in
// order), so a test point's value does not depend on m or on its batch.
constexpr int kTP = 8, kChunk = 4096, kXThreads = 256;

__global__ void __launch_bounds__(kXThreads) cross_partial_kernel(
    const double2* __restrict__ test, int64_t m, const double2* __restrict__ train, int64_t n,
    int metric, double radius, mt_matern th, const double* __restrict__ w,
    double* __restrict__ partial) {
  const int64_t a0 = (int64_t)blockIdx.x * kTP;
  const int64_t lo = (int64_t)blockIdx.y * kChunk;
  const int64_t hi = min(n, lo + kChunk);
  double2 ta[kTP];
  double acc[kTP];
#pragma unroll
  for (int q = 0; q < kTP; ++q) {
    ta[q] = a0 + q < m ? test[a0 + q] : make_double2(0.0, 0.0);
    acc[q] = 0.0;
  }
  for (int64_t b = lo + threadIdx.x; b < hi; b += kXThreads) {
    const double2 pb = train[b];
    const double wb = w[b];
#pragma unroll
    for (int q = 0; q < kTP; ++q) acc[q] += mt_matern_value(dist(ta[q], pb, metric, radius), th) * wb;
  }
  __shared__ double red[kXThreads / 32][kTP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < kTP; ++q) {
    double v = acc[q];
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) red[warp][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < kTP && a0 + threadIdx.x < m) {
    double s = 0.0;
    for (int u = 0; u < kXThreads / 32; ++u) s += red[u][threadIdx.x];
    partial[(int64_t)blockIdx.y * m + a0 + threadIdx.x] = s;
  }
}

__global__ void cross_finish_kernel(const double* __restrict__ partial, int64_t m, int nchunks,
                                    double* __restrict__ out) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < m;
       a += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < nchunks; ++c) s += partial[(int64_t)c * m + a];
    out[a] = s;
  }
}

}  // namespace

int64_t mt_cross_work_doubles_impl(int64_t m, int64_t n) {
  return ((n + kChunk - 1) / kChunk) * (m > 0 ? m : 1);
}

int mt_cross_gemv_impl(const double* test, int64_t m, const double* train, int64_t n, int metric,
                       double radius, const mt_matern& th, const double* w, double* work,
                       double* out, cudaStream_t st) {
  if (m <= 0) return MT_OK;
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  const int64_t mblocks = (m + kTP - 1) / kTP;
  if (nchunks > 65535 || mblocks > (int64_t)INT32_MAX) {
    mt_set_error("cross-covariance product too large (m=%lld, n=%lld)", (long long)m, (long long)n);
    return MT_E_BAD_ARG;
  }
  {
    ProfScope ps(MT_K_MISC, st, 0.0, (double)(m + n) * 16.0 + n * 8.0 + m * 8.0);
    dim3 grid((unsigned)mblocks, (unsigned)nchunks);
    cross_partial_kernel<<<grid, kXThreads, 0, st>>>((const double2*)test, m, (const double2*)train,
                                                     n, metric, radius, th, w, work);
    MT_LAUNCH_CHECK("cross_partial_kernel");
  }
  int64_t blocks = (m + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  cross_finish_kernel<<<(unsigned)blocks, 256, 0, st>>>(work, m, (int)nchunks, out);
  MT_LAUNCH_CHECK("cross_finish_kernel");
  return MT_OK;
}

int mt_generate_impl(const Grid& g, const double* locs, int metric, double radius,
                     const mt_matern& th, cudaStream_t st) {
  const int nrb = (g.nb + kRows - 1) / kRows;
  const int64_t nband = g.nband();
  // grid.x limit 2^31-1: chunk the slot range
  const int64_t max_slots = (int64_t)((1u << 31) - 1) / nrb;
  const double te = (double)g.nb * g.nb;
  for (int64_t s0 = 0; s0 < nband; s0 += max_slots) {
    int64_t cnt = nband - s0 < max_slots ? nband - s0 : max_slots;
    ProfScope ps(MT_K_GEN64, st, 0.0, cnt * te * 8.0);
    gen_kernel<double><<<(unsigned)(cnt * nrb), 256, 0, st>>>(g, (const double2*)locs, metric,
                                                              radius, th, s0, nrb);
    MT_LAUNCH_CHECK("gen_kernel<double>");
  }
  const int64_t noff = g.noff();
  for (int64_t s0 = 0; s0 < noff; s0 += max_slots) {
    int64_t cnt = noff - s0 < max_slots ? noff - s0 : max_slots;
    ProfScope ps(MT_K_GEN32, st, 0.0, cnt * te * 4.0);
    gen_kernel<float><<<(unsigned)(cnt * nrb), 256, 0, st>>>(g, (const double2*)locs, metric,
                                                             radius, th, s0, nrb);
    MT_LAUNCH_CHECK("gen_kernel<float>");
  }
  return MT_OK;
}

int mt_scan_duplicates_impl(const Grid& g, const double* locs, int metric, double radius,
                            cudaStream_t st) {
  int64_t blocks = g.n < 148 * 16 ? g.n : 148 * 16;
  if (blocks < 1) return MT_OK;
  ProfScope ps(MT_K_MISC, st, 0.0, 0.0);
  dup_kernel<<<(unsigned)blocks, 256, 0, st>>>((const double2*)locs, g.n, metric, radius,
                                                g.status);
  MT_LAUNCH_CHECK("dup_kernel");
  return MT_OK;
}

int mt_matern_array_impl(const double* r, int64_t m, const mt_matern& th, double* out,
                         cudaStream_t st) {
  if (m <= 0) return MT_OK;
  int64_t blocks = (m + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  ProfScope ps(MT_K_MISC, st, 0.0, m * 16.0);
  matern_array_kernel<<<(unsigned)blocks, 256, 0, st>>>(r, m, th, out);
  MT_LAUNCH_CHECK("matern_array_kernel");
  return MT_OK;
}
