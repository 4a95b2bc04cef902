// Tile-grid layout shared by every kernel and the host scheduler.
//
// Lower tile grid of an n x n SPD matrix, p = ceil(n/nb) tiles per side,
// tiles nb x nb row-major and padded (identity on the padded diagonal).
// Band tiles (i - j < t) live in an FP64 pool, off-band tiles in an FP32
// pool (MP) or nowhere (DST).  Both pools are ordered column by column
// (tile column j, then tile row i), so panel k and "all trailing tiles of
// step k" are contiguous slot ranges: the panel TRSM and the trailing update
// of a step each launch over one range.  (Reference layout: dict of
// Fortran-ordered tiles, tilestore.py:139-205.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mixtile_b200.h"

#define MT_HD __host__ __device__ __forceinline__

// sum_{x=0}^{n-1} floor((a x + b) / m), a, b >= 0, m > 0 (Euclid-like, O(log))
MT_HD int64_t mt_floor_sum(int64_t n, int64_t m, int64_t a, int64_t b) {
  int64_t ans = 0;
  while (n > 0) {
    if (a >= m) { ans += (n - 1) * n / 2 * (a / m); a %= m; }
    if (b >= m) { ans += n * (b / m); b %= m; }
    const int64_t y = a * n + b;
    if (y < m) break;
    n = y / m;
    b = y % m;
    const int64_t tmp = m; m = a; a = tmp;
  }
  return ans;
}
MT_HD int mt_gcd(int a, int b) { while (b) { const int r = a % b; a = b; b = r; } return a; }

struct Grid {
  int64_t n;
  int nb, p, t, mode;
  double* dp;
  float* sp;
  float* scratch;
  int64_t* status;
  float* split;
  // multi-GPU 2D block-cyclic ownership on a P x Q process grid: this rank
  // stores tiles (i, j) with i = r0 (mod rs) and j = c0 (mod cs), rs = P,
  // cs = Q (single GPU: rs = cs = 1, r0 = c0 = 0)
  int cs = 1, c0 = 0;
  int rs = 1, r0 = 0;
  double* dpanel = nullptr;  // multi-GPU: FP64 rows of the panels in flight (ring)
  // panels in flight in the rings (scratch, split, dpanel): 2 for lookahead 1,
  // 3 for lookahead 2 (panel k is read by the bulk update while k+1 and k+2 form)
  int nring = 2;
  // bulk FP32 update only: SM-yield request word written by the panel stream
  // (cuStreamWriteValue32); CTAs that consume a request exit between work items
  int* yield = nullptr;

  MT_HD int64_t tile_elems() const { return (int64_t)nb * nb; }
  MT_HD bool band(int i, int j) const { return (i - j) < t; }
  MT_HD bool present(int i, int j) const { return mode != MT_MODE_DST || (i - j) < t; }
  MT_HD bool multi() const { return cs > 1 || rs > 1; }
  // logical rows of tile row i (ragged edge, tilestore.py:154-156)
  MT_HD int rows(int i) const {
    int64_t r = n - (int64_t)i * nb;
    return r < nb ? (int)r : nb;
  }
  MT_HD bool owns_col(int j) const { return j >= c0 && (j - c0) % cs == 0; }
  MT_HD bool owns_row(int i) const { return i >= r0 && (i - r0) % rs == 0; }
  MT_HD bool owns(int i, int j) const { return owns_row(i) && owns_col(j); }
  // number of owned tile columns j' < j
  MT_HD int owned_before(int j) const { return j <= c0 ? 0 : (j - c0 + cs - 1) / cs; }
  MT_HD int owned_cols() const { return owned_before(p); }
  MT_HD int owned_col(int m) const { return c0 + m * cs; }
  // owned tile rows i' < x (x >= 0), and the first owned row >= x
  MT_HD int rcnt(int x) const { return rs == 1 ? x : (x - r0 + rs - 1) / rs; }
  MT_HD int first_row(int x) const { return rs == 1 ? x : x + ((r0 - x) % rs + rs) % rs; }
  // sum over owned columns m < mm of rcnt(j_m + d)  (j_m = c0 + m cs)
  MT_HD int64_t rcnt_sum(int mm, int d) const {
    return mt_floor_sum(mm, rs, cs, (int64_t)c0 + d - r0 + rs - 1);
  }

  // first band-pool slot of tile column j: sum over owned j' < j of the owned
  // rows in [j', min(j' + t, p))
  MT_HD int64_t bcol(int j) const {
    const int m = owned_before(j);
    const int m1 = owned_before(p - t + 1);  // owned columns holding t band rows
    if (rs == 1) {
      if (m <= m1) return (int64_t)m * t;
      return (int64_t)m1 * t + (int64_t)(m - m1) * (p - c0) -
             (int64_t)cs * ((int64_t)m * (m - 1) / 2 - (int64_t)m1 * (m1 - 1) / 2);
    }
    const int ma = m < m1 ? m : m1;
    int64_t s = rcnt_sum(ma, t) - rcnt_sum(ma, 0);
    if (m > m1) s += (int64_t)(m - m1) * rcnt(p) - (rcnt_sum(m, 0) - rcnt_sum(m1, 0));
    return s;
  }
  // first off-band-pool slot of tile column j: sum over owned j' < j of the
  // owned rows in [j' + t, p)
  MT_HD int64_t scol(int j) const {
    const int64_t q = p - t;
    if (q <= 0) return 0;
    const int ma = owned_before(j), mb = owned_before((int)q);
    const int mm = ma < mb ? ma : mb;
    if (rs == 1) return (int64_t)mm * (q - c0) - (int64_t)cs * ((int64_t)mm * (mm - 1) / 2);
    return (int64_t)mm * rcnt(p) - rcnt_sum(mm, t);
  }
  MT_HD int64_t nband() const { return bcol(p); }
  MT_HD int64_t noff() const { return mode == MT_MODE_MP ? scol(p) : 0; }
  // pool slot of an owned tile
  MT_HD int64_t dslot(int i, int j) const { return bcol(j) + (rcnt(i) - rcnt(j)); }
  MT_HD int64_t sslot(int i, int j) const { return scol(j) + (rcnt(i) - rcnt(j + t)); }

  // panel ring order (multi-GPU): tile rows grouped by i mod L, L = lcm(P, Q)
  // (1 on a 1 x Q grid), so the rows a process row or column receives are
  // contiguous suffixes of L blocks; single GPU: identity
  MT_HD int ring_l() const { return rs == 1 ? 1 : rs / mt_gcd(rs, cs) * cs; }
  MT_HD int ring_q() const { return (p + ring_l() - 1) / ring_l(); }
  MT_HD int pring() const { return ring_l() * ring_q(); }
  MT_HD int ring_pos(int i) const {
    const int l = ring_l();
    return l == 1 ? i : (i % l) * ring_q() + i / l;
  }
  // multi-GPU panel ring: FP64 rows of panel k (band rows in MP; all in DP)
  MT_HD double* dpanel_tile(int i, int k) const {
    return dpanel + ((int64_t)(k % nring) * pring() + ring_pos(i)) * tile_elems();
  }
  MT_HD int64_t dpanel_row(int i, int k) const {
    return ((int64_t)(k % nring) * pring() + ring_pos(i)) * nb;
  }
  // L_kk for the panel solves: the pool tile on its owner, else the copy
  // broadcast into the FP64 panel ring (row k of panel k)
  MT_HD const double* diag_tile(int k) const {
    return (!multi() || owns(k, k)) ? dtile(k, k) : dpanel_tile(k, k);
  }
  MT_HD double* dtile(int i, int j) const { return dp + dslot(i, j) * tile_elems(); }
  MT_HD float* stile(int i, int j) const { return sp + sslot(i, j) * tile_elems(); }

  // scratch ring: slot s holds [narrowed L_kk][mirrors of band panel rows k+1..k+t-1]
  // (MP, t < p) followed by one tile holding the inverses of L_kk's 32x32 diagonal
  // blocks (FP64, then FP32) used by the panel TRSM
  MT_HD bool has_mirrors() const { return mode == MT_MODE_MP && t < p; }
  MT_HD int nblk32() const { return (nb + 31) / 32; }
  // tiles (of nb*nb floats) holding nblk32 FP64 + FP32 32x32 inverses
  MT_HD int64_t inv_tiles() const {
    const int64_t fl = (int64_t)nblk32() * 1024 * 3;
    return (fl + tile_elems() - 1) / tile_elems();
  }
  MT_HD int64_t slot_tiles() const { return (has_mirrors() ? t : 0) + inv_tiles(); }
  MT_HD float* sslot(int k) const { return scratch + (int64_t)(k % nring) * slot_tiles() * tile_elems(); }
  MT_HD float* sdiag(int k) const { return sslot(k); }
  MT_HD double* sinv64(int k) const {
    return (double*)(sslot(k) + (has_mirrors() ? (int64_t)t : 0) * tile_elems());
  }
  MT_HD float* sinv32(int k) const { return (float*)(sinv64(k) + (int64_t)nblk32() * 1024); }
  // TF32 hi/lo split of FP32 operand (i, k) of panel k (tensor-core engine),
  // ring of two panels in ring order: rows of [hi | lo] per tile row
  MT_HD int64_t split_row(int i, int k) const {
    return ((int64_t)(k % nring) * pring() + ring_pos(i)) * 2 * nb;
  }
  MT_HD float* split_hi(int i, int k) const { return split + split_row(i, k) * nb; }
  MT_HD float* split_lo(int i, int k) const { return split_hi(i, k) + tile_elems(); }
  // split buffer tail (tensor-core TRSM): the pre-TRSM split of the next
  // panel's off-band tiles (written by the update epilogue into column k+1)
  // and the split of W = L_kk^{-1} (row-major), one slot each
  MT_HD int64_t ring_rows() const { return (int64_t)2 * nring * pring(); }  // tile rows
  MT_HD int64_t presplit_row(int i) const { return (ring_rows() + 2 * i) * nb; }
  MT_HD int64_t winv_row() const { return (ring_rows() + 2 * p) * nb; }
  MT_HD int64_t split_rows() const { return (ring_rows() + 2 * p + 2) * nb; }
  MT_HD float* presplit_hi(int i) const { return split + presplit_row(i) * nb; }
  MT_HD float* winv_hi() const { return split + winv_row() * nb; }
  MT_HD float* winv_lo() const { return winv_hi() + tile_elems(); }
  MT_HD float* smirror(int i, int k) const { return sdiag(k) + (int64_t)(i - k) * tile_elems(); }
  // FP32 operand for tile (i,k) of panel k in an FP32 update: payload or mirror
  MT_HD const float* sp_operand(int i, int k) const {
    return band(i, k) ? smirror(i, k) : stile(i, k);
  }

  // slot -> (i, j) inversion by binary search over the owned column starts
  // (a column without owned rows shares its start with the next column, so
  // the largest index with start <= s is a column that holds slot s)
  MT_HD void band_slot_ij(int64_t s, int& i, int& j) const {
    int lo = 0, hi = owned_cols();  // largest owned index m with bcol(col m) <= s
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (bcol(owned_col(mid)) <= s) lo = mid; else hi = mid;
    }
    j = owned_col(lo);
    i = first_row(j) + (int)(s - bcol(j)) * rs;
  }
  MT_HD void off_slot_ij(int64_t s, int& i, int& j) const {
    int lo = 0, hi = owned_before(p - t);
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (scol(owned_col(mid)) <= s) lo = mid; else hi = mid;
    }
    j = owned_col(lo);
    i = first_row(j + t) + (int)(s - scol(j)) * rs;
  }
  __device__ __forceinline__ bool failed() const {
    return *(volatile int64_t*)status >= 0;
  }
};

// ---- L2-friendly output order of the trailing update -----------------------
// Slot order (column by column) re-reads every row operand A_ik from HBM once
// per output column: at p - k = 500 the panel split (2 MB per tile) is far
// larger than L2.  Instead the outputs are visited in super-columns of `sw`
// owned columns, rows ascending inside each, columns ascending inside a row:
// a row operand is then fetched once per super-column and the sw column
// operands stay L2-resident while the rows sweep past.  Every output tile is
// still computed by exactly one work item, so results do not depend on it.
//
// Owned column m is global column j = c0 + m*cs; its off-band rows are
// i in [j + t, p).  In a super-column [ma, mb) row i holds the columns
// m in [ma, min(mb, F(i) + 1)), F(i) = floor((i - t - c0) / cs), so the tiles
// before row x number P(x) = G(x, ma) - G(x, mb) with
// G(x, a) = sum_{i<x} max(0, floor((i - d_a) / cs)), d_a = t + c0 + (a - 1) cs,
// = T(x - d_a) - T(-d_a),  T(Y) = sum_{y<Y} floor(y / cs)  (0 for Y <= 0).
// 32-bit arithmetic: the work-queue owner maps one item per call, and 64-bit
// divisions in a loop over super-columns made that mapping (~10 us per item at
// p = 512) slower than an item's MMA time -- the super-column order then lost
// to slot order (round-2 A/B).  Super-column starts are scol() differences
// (O(1)); one binary search picks the super-column, one the row.
__device__ __forceinline__ int stair_T(int y, int cs) {
  if (y <= 0) return 0;
  const int q = y / cs, r = y - q * cs;
  return cs * (q * (q - 1) / 2) + r * q;
}
__device__ __forceinline__ int stair_G(const Grid& g, int x, int a) {
  const int d = g.t + g.c0 + (a - 1) * g.cs;
  return stair_T(x - d, g.cs) - stair_T(-d, g.cs);
}
__device__ __forceinline__ int super_prefix(const Grid& g, int x, int ma, int mb) {
  return stair_G(g, x, ma) - stair_G(g, x, mb);
}
// tile index -> (i, j) in super-column order over owned columns [mlo, mhi)
// (single process row: rs == 1)
__device__ __forceinline__ void super_tile_ij(const Grid& g, int64_t idx64, int mlo, int mhi, int sw,
                                              int& i, int& j) {
  const int idx = (int)idx64;
  const int base = (int)g.scol(g.owned_col(mlo));
  int lo = 0, hi = (mhi - mlo + sw - 1) / sw;  // largest super-column s starting at <= idx
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if ((int)g.scol(g.owned_col(mlo + mid * sw)) - base <= idx) lo = mid; else hi = mid;
  }
  const int ma = mlo + lo * sw, mb = min(mhi, ma + sw);
  const int local = idx - ((int)g.scol(g.owned_col(ma)) - base);
  int rlo = 0, rhi = g.p;  // largest row x with P(x) <= local
  while (rhi - rlo > 1) {
    const int mid = (rlo + rhi) >> 1;
    if (super_prefix(g, mid, ma, mb) <= local) rlo = mid; else rhi = mid;
  }
  i = rlo;
  j = g.owned_col(ma + (local - super_prefix(g, rlo, ma, mb)));
}


inline Grid make_grid(const mt_tiles* g) {
  Grid r;
  r.n = g->n; r.nb = g->nb; r.p = g->p; r.t = g->t; r.mode = g->mode;
  r.dp = g->dp_pool; r.sp = g->sp_pool; r.scratch = g->scratch; r.status = g->status;
  r.split = g->split;
  r.cs = g->col_stride > 0 ? g->col_stride : 1;
  r.c0 = g->col_offset;
  r.rs = g->row_stride > 0 ? g->row_stride : 1;
  r.r0 = g->row_offset;
  r.nring = g->panel_slots > 2 ? g->panel_slots : 2;
  r.dpanel = g->dpanel;
  return r;
}

// TF32 hi/lo split of an FP32 operand for 3xTF32 products: hi = rna_tf32(x)
// (exact in TF32), lo = x - hi (exact in FP32, so hi + lo == x: the multi-GPU
// DMMA band update rebuilds the FP32 payload from a received split).  The MMA
// reads only lo's TF32 bits; lo's sign is random, so that truncation is
// unbiased.  MT_LO_RNA=1 rounds lo to TF32 instead -- measured on B200
// (tools/acc_tf32.py) to change the factor error by < 1.3x either way, so the
// exact split is kept.
#ifndef MT_LO_RNA
#define MT_LO_RNA 0
#endif
__device__ __forceinline__ void mt_tf32_split(float x, float& hi, float& lo) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  hi = __uint_as_float(h);
  const float r = x - hi;
#if MT_LO_RNA
  uint32_t l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(r));
  lo = __uint_as_float(l);
#else
  lo = r;
#endif
}

// status slots
#define MT_ST_PIVOT 0
#define MT_ST_OVERFLOW 1
#define MT_ST_DUP 2

// error plumbing shared by the translation units
void mt_set_error(const char* fmt, ...);
int mt_cuda_check(cudaError_t e, const char* what);
#define MT_LAUNCH_CHECK(what) \
  do { if (mt_cuda_check(cudaGetLastError(), what)) return MT_E_CUDA; } while (0)

// launch accounting + event profiling (prof.cu)
void mt_count_launch(int n);
int mt_prof_start(int kind, cudaStream_t st, double flops, double bytes);
void mt_prof_stop(int token, cudaStream_t st);
enum MtKind {
  MT_K_GEN64 = 0, MT_K_GEN32, MT_K_POTRF, MT_K_TRSM64, MT_K_TRSM32, MT_K_UPD64, MT_K_UPD32,
  MT_K_SOLVE, MT_K_MISC,
  MT_K_UPD64P, MT_K_UPD32P,  // lookahead panel-column updates (step k -> column k+1)
  MT_NKINDS
};
// device-side span slot [start, end] (ns, %globaltimer) for a kernel that cannot be
// bracketed by stream events; nullptr when not profiling
unsigned long long* mt_prof_dspan(int kind, double flops, double bytes, double share = 1.0);
__device__ __forceinline__ unsigned long long mt_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// brackets the launches of one kernel group with profiling events
struct ProfScope {
  int tok;
  cudaStream_t st;
  ProfScope(int kind, cudaStream_t s, double flops, double bytes, int launches = 1) : st(s) {
    mt_count_launch(launches);
    tok = mt_prof_start(kind, s, flops, bytes);
  }
  ~ProfScope() { mt_prof_stop(tok, st); }
};

// runtime options (api.cu): FP32 update engine and grid cap of the bulk update
// FP32 engines: SIMT FFMA; tcgen05 3xTF32 with round-to-nearest chunk
// accumulation (default, FP32-accurate: tcf_update.cu); tcgen05 3xTF32 with the
// whole K range in TMEM (round-toward-zero accumulation, faster, opt-in)
enum MtEngine { MT_ENGINE_FFMA = 0, MT_ENGINE_TF32X3 = 1, MT_ENGINE_TF32X3_RZ = 2 };
inline bool mt_engine_tc(int e) { return e == MT_ENGINE_TF32X3 || e == MT_ENGINE_TF32X3_RZ; }
int mt_opt_engine();
int mt_opt_update_ctas();
int mt_opt_legacy_dmma();
int mt_opt_pcol_ctas();
int mt_opt_yield_sms();
bool mt_dmma_tma_supported(const Grid& g);
int mt_dmma_update_impl(const Grid& g, int k, int64_t b0, int64_t bcnt, cudaStream_t st,
                        bool pdl = false, unsigned long long* span = nullptr);
int mt_opt_coschedule();
int mt_opt_coschedule_pct();
int mt_opt_potrf_cluster();
int mt_opt_tcf_cluster4();
int mt_opt_tcf_stats();
int mt_opt_tcf_reduce();
bool mt_tc_supported(const Grid& g);
bool mt_tc_trsm_enabled(const Grid& g);  // off-band TRSM as a tcgen05 GEMM against L_kk^{-1}
int mt_tc_trsm_impl(const Grid& g, int k, cudaStream_t st);
int mt_opt_tc_trsm();
int mt_tc_update_impl(const Grid& g, int k, int jlo, int jhi, int ctas, cudaStream_t st,
                      unsigned long long* span = nullptr);
int mt_opt_super_cols();
int mt_opt_wide_items();
int mt_opt_wide_l2pf();
bool mt_tc2w_supported(const Grid& g);
int mt_tc2w_launch(const Grid& g, int k, int64_t s0, int64_t scnt, int ctas, cudaStream_t st,
                   unsigned long long* span);
int mt_tcf_launch(const Grid& g, int k, int64_t s0, int64_t scnt, int ctas, bool trsm, int presplit,
                  cudaStream_t st, unsigned long long* span, int jlo = 0, int jhi = 0);
int mt_tc2_launch(const Grid& g, int k, int64_t s0, int64_t scnt, int ctas, bool trsm,
                  int presplit, cudaStream_t st, unsigned long long* span = nullptr, int jlo = 0,
                  int jhi = 0);
