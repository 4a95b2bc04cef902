// Panel TRSM of step k: A_ik <- A_ik L_kk^{-T} for every present i > k
// (kernels.trsm + factor.py:257-265), batched over the whole panel.
//
//   band rows    (i - k < t): FP64 against L_kk; in MP mode, when a later
//                FP32 update consumes the tile (i + t <= p - 1), the
//                epilogue also writes the RN-narrowed mirror (factor.py:261-262).
//   off-band rows (MP): FP32 against the narrowed L_kk (sp_diag,
//                factor.py:264); the FP64 view is the exact widening and is
//                never materialised (FP64 consumers widen on load).
// Every FP32 operand of this step's FP32 updates also gets its TF32 hi/lo
// split written here (read by the tcgen05 update, tc_update.cu).
//
// Rows of X = B L^{-T} are independent, so a CTA owns RB rows of one tile and
// walks the columns in 32-wide blocks, right-looking:
//   G    = B[:, cb] - X[:, <cb] L[cb, <cb]^T   (thread = 1 column x RB/8 rows;
//          broadcast vector reads of the transposed X, conflict-free reads of L)
//   X_cb = G L_cb,cb^{-T}                      (GEMM against the diagonal-block
//          inverse published by POTRF -- no sequential substitution)
// The 32x32 blocks of L and the inverses are streamed through a 4-stage
// cp.async ring that runs ahead across column blocks.
#include <functional>

#include "mt_grid.cuh"

#define RC_(call) \
  do { int rc__ = (call); if (rc__) return rc__; } while (0)

namespace {

constexpr int kThreads = 256;  // 8 warps; lane = column of the 32-wide block
constexpr int NST = 4;         // cp.async ring depth
constexpr int LDL = 33;        // chunk row stride (conflict-free column reads)

template <typename T> struct Vec;
template <> struct Vec<float> {
  template <int N>
  static __device__ __forceinline__ void ld(const float* p, float (&o)[N]) {
#pragma unroll
    for (int u = 0; u < N; u += 4) {
      float4 v = *(const float4*)(p + u);
      o[u] = v.x; o[u + 1] = v.y; o[u + 2] = v.z; o[u + 3] = v.w;
    }
  }
};
template <> struct Vec<double> {
  template <int N>
  static __device__ __forceinline__ void ld(const double* p, double (&o)[N]) {
#pragma unroll
    for (int u = 0; u < N; u += 2) {
      double2 v = *(const double2*)(p + u);
      o[u] = v.x; o[u + 1] = v.y;
    }
  }
};

template <typename T>
__device__ __forceinline__ void cp_async_elem(T* dst, const T* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "n"(sizeof(T)));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <typename T, int RB>
__global__ void __launch_bounds__(kThreads, 1)
    trsm_kernel(Grid g, int k, int64_t slot0, int nrb, int mirror_ok) {
  if (g.failed()) return;
  constexpr int RPT = RB / 8;                  // rows per thread (4 FP64, 8 FP32)
  constexpr int XS = RB + 16 / sizeof(T);      // Xt row stride (16-byte aligned rows)
  const int64_t slot = slot0 + blockIdx.x / nrb;
  const int rb = blockIdx.x % nrb;
  int i, j;
  const T* L;
  const T* Linv;
  T* B;
  float* M = nullptr;
  if constexpr (sizeof(T) == 8) {
    g.band_slot_ij(slot, i, j);
    L = (const T*)g.diag_tile(k);
    Linv = (const T*)g.sinv64(k);
    B = (T*)g.dtile(i, k);
    if (mirror_ok && g.mode == MT_MODE_MP && i + g.t <= g.p - 1) M = g.smirror(i, k);
  } else {
    g.off_slot_ij(slot, i, j);
    L = (const T*)g.sdiag(k);
    Linv = (const T*)g.sinv32(k);
    B = (T*)g.stile(i, k);
  }
  const int nb = g.nb;
  const int nblk = (nb + 31) / 32;
  const int r0 = rb * RB;
  const int nr = min(RB, nb - r0);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Xt = (T*)smem_raw;                                  // [nblk*32][XS]: Xt[c][r]
  T* ring = Xt + (size_t)nblk * 32 * XS;                 // [NST][32][LDL]
  const int c = threadIdx.x & 31, rw = (threadIdx.x >> 5) * RPT;

  // chunk sequence: for each column block b: L(b, 0..b-1) then inverse(b)
  // chunk index -> (b, q) via b(b+1)/2 + q, q == b meaning "inverse"
  const int nchunks = nblk * (nblk + 1) / 2;
  auto chunk_src = [&](int idx, int& b, int& q) {
    b = (int)((sqrtf(8.0f * idx + 1.0f) - 1.0f) * 0.5f);
    while (b * (b + 1) / 2 > idx) --b;
    while ((b + 1) * (b + 2) / 2 <= idx) ++b;
    q = idx - b * (b + 1) / 2;
  };
  auto issue = [&](int idx) {
    if (idx < nchunks) {
      int b, q;
      chunk_src(idx, b, q);
      T* dst = ring + (size_t)(idx % NST) * 32 * LDL;
      for (int e = threadIdx.x; e < 1024; e += kThreads) {
        const int rr = e >> 5, cc = e & 31;
        const T* src;
        if (q == b) src = Linv + (size_t)b * 1024 + e;     // inverse block, row-major 32x32
        else {
          const int row = min(b * 32 + rr, nb - 1), col = min(q * 32 + cc, nb - 1);
          src = L + (int64_t)row * nb + col;
        }
        cp_async_elem(dst + rr * LDL + cc, src);
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int s = 0; s < NST - 1; ++s) issue(s);

  T acc[RPT];
  int idx = 0;
  for (int b = 0; b < nblk; ++b) {
    const int cb = b * 32, w = min(32, nb - cb);
#pragma unroll
    for (int v = 0; v < RPT; ++v) {
      const int r = rw + v;
      acc[v] = (r < nr && c < w) ? B[(int64_t)(r0 + r) * nb + cb + c] : T(0);
    }
    for (int q = 0; q <= b; ++q, ++idx) {
      cp_async_wait<NST - 2>();
      __syncthreads();
      issue(idx + NST - 1);
      const T* ch = ring + (size_t)(idx % NST) * 32 * LDL;
      if (q < b) {
        // G -= X[:, q-block] L[cb + c, q-block]^T
#pragma unroll 4
        for (int qq = 0; qq < 32; ++qq) {
          T xv[RPT];
          Vec<T>::ld(&Xt[(size_t)(q * 32 + qq) * XS + rw], xv);
          const T l = ch[c * LDL + qq];
#pragma unroll
          for (int v = 0; v < RPT; ++v) acc[v] -= xv[v] * l;
        }
      } else {
        // X_cb = G Linv^T: stage G, then contract with the inverse block
#pragma unroll
        for (int v = 0; v < RPT; ++v) Xt[(size_t)(cb + c) * XS + rw + v] = acc[v];
        __syncthreads();
        T o[RPT];
#pragma unroll
        for (int v = 0; v < RPT; ++v) o[v] = T(0);
#pragma unroll 4
        for (int qq = 0; qq < 32; ++qq) {
          T gv[RPT];
          Vec<T>::ld(&Xt[(size_t)(cb + qq) * XS + rw], gv);
          const T li = ch[c * LDL + qq];
#pragma unroll
          for (int v = 0; v < RPT; ++v) o[v] += gv[v] * li;
        }
        __syncthreads();
#pragma unroll
        for (int v = 0; v < RPT; ++v) Xt[(size_t)(cb + c) * XS + rw + v] = c < w ? o[v] : T(0);
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  // write back; FP32 operands of this step's FP32 updates also get their
  // narrowed mirror (band rows, factor.py:261-262) and, for the tensor-core
  // engine, the TF32 hi/lo split (hi = rna(x), lo = x - hi) read by UMMA
  const bool fp32_operand = (sizeof(T) == 4) || (M != nullptr);
  float* SH = (g.split && fp32_operand) ? g.split_hi(i, k) : nullptr;
  float* SL = SH ? g.split_lo(i, k) : nullptr;
  double* DP = (sizeof(T) == 8 && g.multi() && g.dpanel) ? g.dpanel_tile(i, k) : nullptr;
  for (int r = threadIdx.x >> 5; r < nr; r += kThreads / 32) {
    for (int cc = c; cc < nb; cc += 32) {
      const T v = Xt[(size_t)cc * XS + r];
      const int64_t o = (int64_t)(r0 + r) * nb + cc;
      B[o] = v;
      const float f = __double2float_rn((double)v);
      if (M) M[o] = f;
      if (DP) DP[o] = (double)v;  // multi-GPU: FP64 band panel row for the broadcast
      if (SH) {
        float h, l;
        mt_tf32_split(f, h, l);
        SH[o] = h;
        SL[o] = l;
      }
    }
  }
}

template <typename T, int RB>
size_t trsm_smem(int nb) {
  const size_t rows = (size_t)((nb + 31) / 32) * 32;
  return (rows * (RB + 16 / sizeof(T)) + (size_t)NST * 32 * LDL) * sizeof(T);
}

template <typename T, int RB>
int launch_trsm(const Grid& g, int k, int64_t s0, int64_t cnt, int mirror_ok, cudaStream_t st) {
  if (cnt <= 0) return MT_OK;
  const int nrb = (g.nb + RB - 1) / RB;
  const size_t smem = trsm_smem<T, RB>(g.nb);
  cudaFuncSetAttribute(trsm_kernel<T, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  const double rk = g.rows(k), nb = g.nb;
  // algorithmic work: rows(i) * rows(k)^2 per tile (factor.py:88-90); last row may be ragged
  const bool last = (sizeof(T) == 8 ? (k + g.t >= g.p) : true) && cnt > 0;
  const double rows_sum = (cnt - (last ? 1 : 0)) * nb + (last ? g.rows(g.p - 1) : 0);
  ProfScope ps(sizeof(T) == 8 ? MT_K_TRSM64 : MT_K_TRSM32, st, rows_sum * rk * rk,
               cnt * nb * nb * sizeof(T) * 2.0);
  trsm_kernel<T, RB><<<(unsigned)(cnt * nrb), kThreads, smem, st>>>(g, k, s0, nrb, mirror_ok);
  MT_LAUNCH_CHECK("trsm_kernel");
  return MT_OK;
}

// W = L_kk^{-1} (lower, FP64) for the tensor-core off-band TRSM X = B W^T.
// The columns of W are independent triangular solves L w_c = e_c, so CTA b
// owns the 8 columns c0 = 8b .. c0+7 (64 CTAs at nb = 512: a short dependent
// chain per CTA) and walks their 32-row blocks down:
//   W[cb, cols] = Li_cb[:, cols]            (POTRF's diagonal-block inverse)
//   W[rb, cols] = -Li_rb (L[rb, cb:rb] W[cb:rb, cols])
// Both products run on DMMA (m8n8k4 f64, one 8 x 8 fragment per warp).  The L
// row blocks and Li_rb do not depend on W: they stream through a 4-deep
// cp.async ring of 32 x 64 chunks ahead of the dependent chain.  The result is
// written row-major as its FP32 rounding split into TF32 hi/lo (the operand
// format of the 3xTF32 UMMA), zeros above the diagonal.
constexpr int TW = 8;     // columns of W per CTA
constexpr int CW = 64;    // chunk width (columns of L)
constexpr int CLD = 68;   // chunk row stride (doubles): 16-B rows, 2-wavefront fragments
constexpr int NCH = 4;    // ring depth

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src));
}
__device__ __forceinline__ void dmma_884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(128) trinv_kernel(Grid g, int k) {
  if (g.failed()) return;
  const int nb = g.nb, nblk = nb / 32;
  const int c0 = blockIdx.x * TW, cb = c0 / 32, cc0 = c0 % 32;
  const double* __restrict__ L = g.dtile(k, k);
  const double* __restrict__ inv = g.sinv64(k);
  extern __shared__ __align__(16) double wsm[];
  double* Wc = wsm;                 // [nb][TW]: columns c0.. of W (rows >= cb*32 used)
  double* Tt = Wc + nb * TW;        // [32][TW]
  double* ring = Tt + 32 * TW;      // [NCH][32][CLD]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fr = lane >> 2, fk = lane & 3;

  // chunk sequence: for rb = cb+1.., L chunks q0 = cb*32, +64, .. < rb*32, then Li_rb
  auto chunk_of = [&](int idx, int& rb, int& q0) {
    for (rb = cb + 1; rb < nblk; ++rb) {
      const int n = (rb - cb + 1) / 2 + 1;
      if (idx < n) {
        q0 = idx == n - 1 ? -1 : cb * 32 + idx * CW;
        return true;
      }
      idx -= n;
    }
    return false;
  };
  auto issue = [&](int idx) {
    int rb, q0;
    if (chunk_of(idx, rb, q0)) {
      double* dst = ring + (idx % NCH) * 32 * CLD;
      if (q0 < 0) {  // Li_rb, 32 x 32 row-major
        for (int e = tid; e < 32 * 16; e += 128) {
          const int rr = e >> 4, c = (e & 15) * 2;
          cp_async16(dst + rr * CLD + c, inv + rb * 1024 + rr * 32 + c);
        }
      } else {
        const int hw = min(CW, rb * 32 - q0) / 2;
        for (int e = tid; e < 32 * hw; e += 128) {
          const int rr = e / hw, c = (e % hw) * 2;
          cp_async16(dst + rr * CLD + c, L + (int64_t)(rb * 32 + rr) * nb + q0 + c);
        }
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
#pragma unroll
  for (int c = 0; c < NCH - 1; ++c) issue(c);

  for (int e = tid; e < 32 * TW; e += 128) {  // diagonal block: columns of Li_cb
    const int rr = e / TW, c = e % TW;
    Wc[(cb * 32 + rr) * TW + c] = inv[cb * 1024 + rr * 32 + cc0 + c];
  }
  int idx = 0;
  for (int rb = cb + 1; rb < nblk; ++rb) {
    // T (32 x 8) = L[rb, cb:rb] W[cb:rb, cols]: warp w owns rows 8w..8w+7
    double acc[2] = {0.0, 0.0};
    for (int q0 = cb * 32; q0 < rb * 32; q0 += CW, ++idx) {
      asm volatile("cp.async.wait_group %0;\n" ::"n"(NCH - 2));
      __syncthreads();  // chunk idx landed; the slot of idx-1 is free
      issue(idx + NCH - 1);
      const double* ch = ring + (idx % NCH) * 32 * CLD + (warp * 8 + fr) * CLD + fk;
      const double* wb = Wc + (q0 + fk) * TW + fr;
      const int w = min(CW, rb * 32 - q0);
#pragma unroll 4
      for (int k4 = 0; k4 < w; k4 += 4) dmma_884(acc, ch[k4], wb[k4 * TW]);
    }
    Tt[(warp * 8 + fr) * TW + 2 * fk] = acc[0];
    Tt[(warp * 8 + fr) * TW + 2 * fk + 1] = acc[1];
    asm volatile("cp.async.wait_group %0;\n" ::"n"(NCH - 2));
    __syncthreads();  // T complete; Li_rb landed
    issue(idx + NCH - 1);
    const double* li = ring + (idx % NCH) * 32 * CLD + (warp * 8 + fr) * CLD + fk;
    ++idx;
    double o[2] = {0.0, 0.0};
#pragma unroll
    for (int k4 = 0; k4 < 32; k4 += 4) dmma_884(o, li[k4], Tt[(k4 + fk) * TW + fr]);
    Wc[(rb * 32 + warp * 8 + fr) * TW + 2 * fk] = -o[0];
    Wc[(rb * 32 + warp * 8 + fr) * TW + 2 * fk + 1] = -o[1];
    __syncthreads();  // W_rb visible; Tt reusable
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  float* WH = g.winv_hi();
  float* WL = g.winv_lo();
  for (int e = tid; e < nb * TW; e += 128) {
    const int R = e / TW, c = e % TW;
    const double w = R >= cb * 32 ? Wc[R * TW + c] : 0.0;
    const float f = __double2float_rn(w);
    float h, l;
    mt_tf32_split(f, h, l);
    const int64_t o = (int64_t)R * nb + c0 + c;
    WH[o] = h;
    WL[o] = l;
  }
}

// pre-TRSM split of panel k's off-band tiles (k = 0, or when no update
// epilogue produced it): presplit(i) = {rna_tf32(x), x - hi}
__global__ void __launch_bounds__(256) presplit_kernel(Grid g, int k, int64_t s0) {
  const int64_t te = g.tile_elems();
  const int64_t slot = s0 + blockIdx.y;
  int i, j;
  g.off_slot_ij(slot, i, j);
  const float4* src = (const float4*)g.stile(i, k);
  float4* hi = (float4*)g.presplit_hi(i);
  float4* lo = (float4*)(g.presplit_hi(i) + te);
  for (int64_t e = blockIdx.x * 256 + threadIdx.x; e < te / 4; e += (int64_t)gridDim.x * 256) {
    const float4 x = src[e];
    float4 h, l;
    float* xp = (float*)&x;
    float* hp = (float*)&h;
    float* lp = (float*)&l;
#pragma unroll
    for (int u = 0; u < 4; ++u) mt_tf32_split(xp[u], hp[u], lp[u]);
    hi[e] = h;
    lo[e] = l;
  }
}

}  // namespace

int mt_trinv_impl(const Grid& g, int k, cudaStream_t st) {
  const size_t smem = ((size_t)g.nb * TW + 32 * TW + (size_t)NCH * 32 * CLD) * sizeof(double);
  cudaFuncSetAttribute(trinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const double nb = g.nb;
  ProfScope ps(MT_K_MISC, st, nb * nb * nb / 3.0, nb * nb * 16.0);
  trinv_kernel<<<g.nb / TW, 128, smem, st>>>(g, k);
  MT_LAUNCH_CHECK("trinv_kernel");
  return MT_OK;
}

int mt_presplit_impl(const Grid& g, int k, cudaStream_t st) {
  const int64_t s0 = g.scol(k), cnt = g.scol(k + 1) - s0;
  if (cnt <= 0) return MT_OK;
  ProfScope ps(MT_K_MISC, st, 0.0, cnt * (double)g.tile_elems() * 12.0);
  presplit_kernel<<<dim3(16, (unsigned)cnt), 256, 0, st>>>(g, k, s0);
  MT_LAUNCH_CHECK("presplit_kernel");
  return MT_OK;
}

// Panel rows i in (k, p) of tile column k that this rank stores.  Band rows:
// the band slots of column k after the diagonal tile (when it is ours);
// off-band rows: off slots scol(k) .. scol(k+1)-1.  On a multi-GPU grid
// W = L_kk^{-1} is formed by the diagonal tile's owner (mt_panel_factor) and
// broadcast down the process column with L_kk and its 32x32 inverses.
int mt_trsm_impl(const Grid& g, int k, cudaStream_t st, const std::function<int()>* before) {
  auto pre = [&]() { return before ? (*before)() : MT_OK; };
  if (trsm_smem<double, 32>(g.nb) > 220 * 1024 || trsm_smem<float, 64>(g.nb) > 220 * 1024) {
    mt_set_error("trsm: nb=%d too large for the shared-memory panel", g.nb);
    return MT_E_BAD_ARG;
  }
  RC_(pre());
  const int64_t b0 = g.bcol(k) + (g.owns(k, k) ? 1 : 0);
  int rc = launch_trsm<double, 32>(g, k, b0, g.bcol(k + 1) - b0, 1, st);
  if (rc) return rc;
  if (g.mode == MT_MODE_MP && g.scol(k + 1) > g.scol(k)) {
    if (mt_tc_trsm_enabled(g)) {
      // the update epilogue of step k-1 pre-split column k (k = 0: nobody did)
      if (k == 0) RC_(mt_presplit_impl(g, k, st));
      if (!g.multi()) {
        RC_(pre());
        RC_(mt_trinv_impl(g, k, st));
      }
      RC_(pre());
      rc = mt_tc_trsm_impl(g, k, st);
    } else {
      rc = launch_trsm<float, 64>(g, k, g.scol(k), g.scol(k + 1) - g.scol(k), 0, st);
    }
  }
  return rc;
}
