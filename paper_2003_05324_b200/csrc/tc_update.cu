// FP32 (off-band) trailing update and off-band panel TRSM on the 5th-gen
// tensor cores: 3xTF32, dispatch between the engines, and the host-side TMA
// tensor-map encoding shared by every TMA kernel.
//
//   C_ij <- C_ij - A_ik A_jk^T      (kernels.gemm FP32 path, factor.py:273-274)
//
// FP32 products are emulated with three TF32 UMMAs per K-step,
//   A B^T ~= A_lo B_hi^T + A_hi B_lo^T + A_hi B_hi^T,
// hi = cvt.rna.tf32(x) (exactly representable in TF32), lo = x - hi (exact
// in FP32; Grid-level helper mt_tf32_split).  The dropped A_lo B_lo term and
// the TF32 truncation of lo are O(2^-22) relative.  The hi/lo split is
// produced once per panel tile by the TRSM epilogue (Grid::split_hi/lo), so
// the updates stream both halves straight from L2 with TMA.
//
// Engines: tcf_update.cu (default; TMEM accumulator flushed into
// round-to-nearest FP32 sums every 32 K-columns -- FP32-accurate) and the
// opt-in whole-K engines tc2w_update.cu / tc2_update.cu (TMEM accumulation
// rounds toward zero).  Every output element is written by one CTA pair per
// step in ascending k: deterministic, schedule-invariant.
#include <cuda.h>

#include "tma.cuh"

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
  return g.mode == MT_MODE_MP && g.split != nullptr && g.nb % 256 == 0 &&
         g.split_rows() < (1ll << 31);
}

bool mt_tc_trsm_enabled(const Grid& g) {
  return mt_opt_tc_trsm() && (mt_engine_tc(mt_opt_engine()) || g.multi()) &&
         mt_tc_supported(g);
}

namespace {
// launch over `nitems` work items of slot range [s0, s0 + scnt)
int launch_tc32(const Grid& g, int k, int64_t s0, int64_t scnt, int ctas, bool trsm,
                cudaStream_t st, int jlo = 0, int jhi = 0, unsigned long long* span = nullptr) {
  if (scnt <= 0) return MT_OK;
  const int presplit = (!trsm && mt_tc_trsm_enabled(g)) ? 1 : 0;
  // default engine: round-to-nearest chunked accumulation (tcf_update.cu)
  if (mt_opt_engine() != MT_ENGINE_TF32X3_RZ)
    return mt_tcf_launch(g, k, s0, scnt, ctas, trsm, presplit, st, span, jlo, jhi);
  // opt-in engine 2: whole K range in TMEM; 256 x 512 CTA-pair items for the
  // bulk update (tc2w_update.cu), 256 x 256 items otherwise (tc2_update.cu)
  if (!trsm && mt_opt_wide_items() && mt_tc2w_supported(g) && jlo > k + 1)
    return mt_tc2w_launch(g, k, s0, scnt, ctas, st, span);
  return mt_tc2_launch(g, k, s0, scnt, ctas, trsm, presplit, st, span, jlo, jhi);
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
