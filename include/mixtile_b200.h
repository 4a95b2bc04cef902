/*
 * mixtile_b200 -- C ABI of the B200-native mixed-precision tile-Cholesky
 * Gaussian log-likelihood (arXiv 2003.05324), drop-in for the reference
 * package `mixtile`'s hot path.
 *
 * Every entry point takes plain pointers and sizes.  Device pointers are
 * allocated by the caller (the Python host uses torch's caching allocator);
 * `stream` is a cudaStream_t passed as void*.  All calls are asynchronous on
 * `stream` unless documented otherwise; `mt_read_status` synchronises.
 * Return value: MT_OK, or an MT_E* code with details in mt_last_error().
 *
 * The reference interfaces each entry replaces (paths under the reference's
 * pkg/src/mixtile/) are cited per function.
 */
#ifndef MIXTILE_B200_H
#define MIXTILE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: map 1:1 onto the reference's exception types */
#define MT_OK 0
#define MT_E_NOT_SPD 1      /* factor.FactorizationError(index)       factor.py:31-37  */
#define MT_E_OVERFLOW 2     /* tilestore.PrecisionOverflowError       tilestore.py:20  */
#define MT_E_BAD_ARG 3      /* ValueError                                               */
#define MT_E_CUDA 4         /* RuntimeError (CUDA/NCCL failure)                         */

/* precision modes (tilestore.Mode, tilestore.py:24-27) */
#define MT_MODE_DP 0
#define MT_MODE_MP 1
#define MT_MODE_DST 2

/* distance metrics (covmath.DistanceMetric, covmath.py:299-317) */
#define MT_METRIC_EUCLIDEAN 0
#define MT_METRIC_GREAT_CIRCLE 1

/*
 * Device-resident lower tile grid of an n x n symmetric matrix
 * (replaces tilestore.TileMatrix, tilestore.py:139-205).
 *
 * Tiles are nb x nb, ROW-major, padded: the last tile row/column is padded
 * to nb with identity on the diagonal and zeros elsewhere, which leaves the
 * factor, logdet and solves of the n x n problem unchanged.  Tile (i,j),
 * i >= j, is "band" iff i - j < t (tilestore.band_member, tilestore.py:92-96).
 *   dp_pool: band tiles, FP64, column-major tile order (column j, then row i).
 *   sp_pool: off-band tiles, FP32 (MP only), same order.
 *   scratch: panel scratch, mt_scratch_tiles(p, t, mode, nb) FP32-sized tiles, a ring of
 *            two slots: [narrowed L_kk][narrowed band-panel mirrors] (MP,
 *            factor.py:255,262) + one tile holding the inverses of L_kk's
 *            32x32 diagonal blocks (FP64 and FP32) for the panel TRSM.
 *   status:  int64[4] device: [0] first failing global pivot (-1 = none),
 *            [1] FP32 narrowing overflow count, [2] duplicate-location pairs.
 *   split:   TF32 hi/lo split of panels k (ring of 2): tile (i, k) of panel k at
 *            split + ((k&1)*pr + ring(i))*2*nb*nb (hi) and + nb*nb (lo), pr = p
 *            and ring(i) = i on one GPU (see row_stride below); then the
 *            pre-TRSM split of the next panel's off-band tiles at
 *            split + (4pr + 2i)*nb*nb, and the split of W = L_kk^{-1} (row-major)
 *            at split + (4pr + 2p)*nb*nb (hi) / + nb*nb (lo): 6p + 2 tiles on
 *            one GPU (mt_split_tiles), mt_split_tiles_ex() on a P x Q grid.
 */
typedef struct mt_tiles {
  int64_t n;
  int32_t nb;
  int32_t p;     /* ceil(n / nb) */
  int32_t t;     /* resolved band thickness; p in DP mode */
  int32_t mode;  /* MT_MODE_* */
  double* dp_pool;
  float* sp_pool;
  float* scratch;
  int64_t* status;
  float* split;  /* optional (MP, tensor-core engine): mt_split_tiles() FP32 tiles holding
                    the TF32 hi/lo split of the two panels in flight; NULL disables the
                    tcgen05 3xTF32 update (FFMA fallback kernel is used instead) */
  /* multi-GPU, 2D block-cyclic over a P x Q process grid: this rank stores
   * only the tiles (i, j) with j = col_offset (mod col_stride = Q) and
   * i = row_offset (mod row_stride = P), column by column, rows ascending;
   * strides 1 and offsets 0 are the single-GPU layout.  dpanel:
   * mt_dpanel_tiles_ex() FP64 tiles receiving the FP64 rows of the two panels
   * in flight (NULL on a single GPU).  Panel rings (split, dpanel) are in
   * "ring order" on a multi-GPU grid: tile row i at position
   * (i mod L) * ceil(p / L) + i / L, L = lcm(P, Q) (L = 1 when P = 1), so the
   * rows one process row or column receives are contiguous. */
  int32_t col_stride;
  int32_t col_offset;
  double* dpanel;
  int32_t row_stride;
  int32_t row_offset;
  /* panels in flight in the scratch / split / dpanel rings: 0 or 2 (lookahead
   * 1), 3 (lookahead 2); sizes from mt_ring_tiles() */
  int32_t panel_slots;
} mt_tiles;

/* Matern parameters + per-theta Bessel constants (covmath.py:72-95, 228-283),
 * filled on the host by mt_matern_prepare(). */
typedef struct mt_matern {
  double variance, spatial_range, smoothness;
  int32_t kind;      /* 0: nu = 0.5 closed form, 1: nu = 1.5 closed form, 2: Bessel */
  int32_t nl;        /* int(nu + 1/2) upward recurrences */
  double mu;         /* nu - nl, in [-1/2, 1/2] */
  double gam1, gam2; /* Temme gammas */
  double rp, rm;     /* 1/Gamma(1+mu), 1/Gamma(1-mu) */
  double fact;       /* 1/sinc(mu) */
  double scale;      /* variance 2^(1-nu) / Gamma(nu) */
} mt_matern;

/* sizes of the pools for a layout (element counts are tiles * nb * nb) */
int64_t mt_dp_tiles(int32_t p, int32_t t, int32_t mode);
int64_t mt_sp_tiles(int32_t p, int32_t t, int32_t mode);
int64_t mt_scratch_tiles(int32_t p, int32_t t, int32_t mode, int32_t nb);
int64_t mt_split_tiles(int32_t p, int32_t t, int32_t mode);
int32_t mt_version(void);
const char* mt_last_error(void);

/* Covariance tile generation: FP64 band tiles, FP32 off-band tiles written
 * directly, DST off-band tiles absent; padding set.  Overflow of a finite
 * value on narrowing increments status[1].
 * Replaces TileAssembler.assemble / assemble_covariance (tilestore.py:243-262).
 * locs: device, n x 2 row-major FP64. */
int mt_generate(const mt_tiles* g, const double* locs, int32_t metric, double radius,
                const mt_matern* theta, void* stream);

/* Duplicate-location scan: status[2] += #pairs a<b with distance == 0
 * (TileAssembler.__init__, tilestore.py:225-241). */
int mt_scan_duplicates(const mt_tiles* g, const double* locs, int32_t metric, double radius,
                       void* stream);

/* Matern covariance at m distances (covmath.matern_array, covmath.py:261-283). */
int mt_matern_array(const double* r, int64_t m, const mt_matern* theta, double* out,
                    void* stream);

/* Kriging cross-covariance product (predict.krige, predict.py:37-49: the
 * `matern_array(pairwise_distance(test, train)) @ weights` step), fused so the
 * m x n cross-covariance is never stored:
 *   out[a] = sum_b C(d(test_a, train_b)) w[b],  a < m, b < n,
 * FP64, fixed reduction order.  test (m x 2), train (n x 2), w (n), out (m):
 * device; work: mt_cross_work_doubles(m, n) device doubles. */
int64_t mt_cross_work_doubles(int64_t m, int64_t n);
int mt_cross_gemv(const double* test, int64_t m, const double* train, int64_t n, int32_t metric,
                  double radius, const mt_matern* theta, const double* w, double* work,
                  double* out, void* stream);

/* Band-precision tile Cholesky in place (factor.cholesky, factor.py:230-285):
 * POTRF/TRSM/SYRK/GEMM right-looking with `lookahead` (0 or 1) on a private
 * high-priority panel stream joined back to `stream`.  A non-positive pivot
 * sets status[0] to the global 0-based index (FactorizationError.index). */
int mt_cholesky(const mt_tiles* g, int32_t lookahead, void* stream);

/* mt_cholesky with the forward sweep of mt_quad fused into the schedule (each
 * column's TRSV/GEMV step issued as soon as the column is final, underneath the
 * bulk updates): factors in place and writes quad = ||L^{-1} z||^2 to *out
 * (device), bitwise equal to mt_cholesky + mt_quad.  work: mt_work_doubles(). */
int mt_cholesky_quad(const mt_tiles* g, int32_t lookahead, const double* z, double* work,
                     double* out, void* stream);

/* Device scratch (doubles) needed by mt_logdet / mt_quad / mt_evaluate:
 * p*nb + 2048 + p. */
int64_t mt_work_doubles(const mt_tiles* g);

/* log det = 2 sum log diag(L) (factor.logdet, factor.py:318-323) -> *out (device);
 * work: >= p device doubles. */
int mt_logdet(const mt_tiles* g, double* work, double* out, void* stream);

/* In-place solves on device rhs x (n_pad x nrhs row-major, n_pad = p*nb,
 * rows >= n must be zero): which = 1 forward L y = b, 2 backward L^T x = y,
 * 3 both (factor.solve, factor.py:292-315). */
int mt_solve(const mt_tiles* g, double* x, int64_t nrhs, int32_t which, void* stream);

/* quad = z^T (L L^T)^{-1} z = ||L^{-1} z||^2 by the forward sweep only;
 * z: device n_pad doubles (zero padded); work: mt_work_doubles() device
 * doubles; *out (device). (mle._evaluate, mle.py:80-86) */
int mt_quad(const mt_tiles* g, const double* z, double* work, double* out, void* stream);

/* out = L v (factor.matvec_lower, factor.py:326-340); v, out device n_pad. */
int mt_matvec_lower(const mt_tiles* g, const double* v, double* out, void* stream);

/* One fused likelihood evaluation: generate -> cholesky -> logdet -> quad.
 * out2 (device): [logdet, quad]; work: mt_work_doubles() device doubles.
 * The caller resets status before and reads it after (mt_read_status).
 * (mle._evaluate, mle.py:80-86) */
int mt_evaluate(const mt_tiles* g, const double* locs, int32_t metric, double radius,
                const mt_matern* theta, const double* z, double* work, double* out2,
                int32_t lookahead, void* stream);

/* ---- multi-GPU factorization, one process per GPU, 2D block-cyclic over a
 * P x Q grid (row_stride = P, col_stride = Q; rank (r, c) stores tiles with
 * i = r mod P, j = c mod Q).  The host drives the step loop: POTRF(k) on the
 * owner of (k, k); on P > 1 L_kk, its 32x32 inverses and W = L_kk^{-1}
 * (mt_diag_regions) go down process column k mod Q; TRSM(k) on that column's
 * ranks; panel k's rows (split hi/lo + FP64 rows in dpanel, ring order) are
 * broadcast along process rows, then down process columns.  Every tile keeps
 * the single-GPU update order: the factor is bitwise identical for any grid. */
/* POTRF(k) + TRSM(k) of the owned tile column k on a 1 x Q grid (factor.py:249-265). */
int mt_panel(const mt_tiles* g, int32_t k, void* stream);
/* POTRF(k) on the owner of (k, k) (+ L_kk into dpanel, W split, on a grid). */
int mt_panel_factor(const mt_tiles* g, int32_t k, void* stream);
/* TRSM(k) of this rank's rows of tile column k. */
int mt_panel_solve(const mt_tiles* g, int32_t k, void* stream);
/* {offset, count} of L_kk in dpanel (doubles), of its 32x32 inverses in scratch
 * (floats) and of W's split in split (floats): the column broadcast of panel k. */
int mt_diag_regions(const mt_tiles* g, int32_t k, int64_t* out6);
/* Step-k trailing updates of the owned columns in [jlo, jhi) (factor.py:266-274);
 * panel k must be present in split/dpanel. */
int mt_update(const mt_tiles* g, int32_t k, int32_t jlo, int32_t jhi, void* stream);
/* mt_update with flags: bit 0 = this (bulk) update may yield SMs between work
 * items when mt_yield_request() posts a request (the caller's panel stream
 * then gets them for POTRF/TRSM and the broadcast). */
int mt_update_ex(const mt_tiles* g, int32_t k, int32_t jlo, int32_t jhi, int32_t flags,
                 void* stream);
/* Post (in `stream` order, no SM needed: cuStreamWriteValue32) a request that
 * running yield-enabled bulk updates release `sms` SMs; 0 withdraws it.
 * No-op when stream memory operations are unavailable. */
int mt_yield_request(int32_t sms, void* stream);
/* partial[k] = sum log diag(L_kk) for owned k, 0 otherwise (factor.py:318-323). */
int mt_logdet_partials(const mt_tiles* g, double* partial, void* stream);
/* Forward-sweep step i on the owner of column i: y_i = L_ii^{-1} x_i, x_r -= L_ri y_i. */
int mt_fwd_step(const mt_tiles* g, int32_t i, double* x, void* stream);
/* The same split by owner: which bit 0 = y_i = L_ii^{-1} x_i (owner of (i, i)),
 * bit 1 = x_r -= L_ri y_i for this rank's rows r > i (ranks of column i). */
int mt_fwd_step_ex(const mt_tiles* g, int32_t i, int32_t which, double* x, void* stream);
/* Sum of squares of m device doubles with mt_quad's fixed-order reduction
 * (work: >= 1024 device doubles) -> *out (device). */
int mt_sumsq(const double* x, int64_t m, double* work, double* out, void* stream);
/* Local pool sizes (tiles) of a rank's columns (1 x Q grid); dpanel ring size. */
int mt_local_tiles(int32_t p, int32_t t, int32_t mode, int32_t col_stride, int32_t col_offset,
                   int64_t* ndp, int64_t* nsp);
int64_t mt_dpanel_tiles(int32_t p, int32_t t, int32_t mode);
/* The same on a P x Q grid for rank (row_offset, col_offset); ring sizes. */
int mt_local_tiles_ex(int32_t p, int32_t t, int32_t mode, int32_t row_stride, int32_t row_offset,
                      int32_t col_stride, int32_t col_offset, int64_t* ndp, int64_t* nsp);
int64_t mt_dpanel_tiles_ex(int32_t p, int32_t row_stride, int32_t col_stride);
int64_t mt_split_tiles_ex(int32_t p, int32_t t, int32_t mode, int32_t row_stride,
                          int32_t col_stride);
/* Ring-buffer sizes (tiles) for `slots` panels in flight (2: lookahead 1,
 * 3: lookahead 2) on a P x Q grid: scratch (FP32 tiles), split (FP32 tiles,
 * 0 when the layout has no FP32 operands), dpanel (FP64 tiles, multi-GPU). */
int mt_ring_tiles(int32_t p, int32_t t, int32_t mode, int32_t nb, int32_t row_stride,
                  int32_t col_stride, int32_t slots, int64_t* scratch, int64_t* split,
                  int64_t* dpanel);
/* Ring position of tile row i on a P x Q grid (see mt_tiles.row_stride). */
int32_t mt_ring_pos(int32_t p, int32_t row_stride, int32_t col_stride, int32_t i);

/* Diagnostics (option 16 = 1): {MMA-issuer cycles waiting for operands, for a
 * drained TMEM chunk, total issuer cycles, issuers} of the FP32 tcgen05 update
 * since the last call (then reset). */
int mt_tcf_stats(double* out4);

/* Synchronise `stream` and read status: *bad_pivot (-1 none), *overflow,
 * *duplicates.  Returns MT_E_NOT_SPD / MT_E_OVERFLOW when set, else MT_OK. */
int mt_read_status(const mt_tiles* g, int64_t* bad_pivot, int64_t* overflow,
                   int64_t* duplicates, void* stream);

/* Reset status to {-1, 0, 0, 0} (async). */
int mt_reset_status(const mt_tiles* g, void* stream);

/* Tile transfer for the host view and TileMatrix.from_dense (tilestore.py:167-205):
 * which = 0 FP64 payload (band pool), 1 FP32 payload (off-band pool).
 * Host buffers are rows x cols COLUMN-major (numpy Fortran order, the
 * reference's tile layout); rows/cols = logical (unpadded) tile shape. */
int mt_get_tile(const mt_tiles* g, int32_t i, int32_t j, int32_t which, void* host, void* stream);
int mt_put_tile(const mt_tiles* g, int32_t i, int32_t j, int32_t which, const void* host,
                void* stream);

/* Host-buffer end-to-end evaluation (the FFI-facing call): allocates device
 * memory, copies locs (n x 2) and z (n) in, runs mt_evaluate, copies
 * [logdet, quad] out, frees.  Returns MT_E_NOT_SPD with *bad_pivot set on an
 * indefinite covariance. (mle.loglik, mle.py:89-99 minus the final affine) */
int mt_evaluate_host(int64_t n, int32_t nb, int32_t mode, int32_t t, const double* locs,
                     const double* z, int32_t metric, double radius, const mt_matern* theta,
                     double* out2, int64_t* bad_pivot);

/* --- tracing (the reference records wall time only, cli.py:253-258) ---
 * mt_launch_count: kernels launched by this library since load.
 * mt_prof_begin/end: bracket every launch group with CUDA events on its own
 * stream; end() synchronises the device and returns, per kernel kind
 * (0 gen64, 1 gen32, 2 potrf, 3 trsm64, 4 trsm32, 5 upd64, 6 upd32, 7 solve,
 * 8 misc), total device ms, algorithmic flops, algorithmic bytes, launches. */
long long mt_launch_count(void);
int mt_prof_begin(int32_t capacity);
int mt_prof_end(int32_t nkinds, double* ms, double* flops, double* bytes, int64_t* count);
/* After mt_prof_end: per kind, sum of ms x (fraction of the SMs each launch was
 * given).  Launches that overlap another kernel by design (the FP32 bulk update
 * co-scheduled with the band update, option 10) time themselves on the device
 * (%globaltimer spans) and run on a share of the SMs. */
int mt_prof_sm_weighted(int32_t nkinds, double* ms_w);

/* Peak probes for roofline denominators: kind 0 FFMA, 1 DFMA, 2 FP64 DMMA;
 * *tflops = achieved TFLOP/s of a dependent-chain FMA kernel on all SMs. */
int mt_peak_probe(int32_t kind, int32_t iters, double* tflops);

/* Runtime options; returns the previous value.
 *   0: FP32 (off-band) update engine: 0 = SIMT FFMA, 1 = tcgen05 3xTF32 with
 *      round-to-nearest chunk accumulation (default), 2 = tcgen05 3xTF32 with
 *      whole-K TMEM accumulation (round-toward-zero; faster, opt-in)
 *   1: CTA cap of the bulk trailing update (0 = all SMs)
 *   2: 1 = register-staged DMMA band update instead of the TMA-staged one
 *   3: off-band panel TRSM: 1 = tcgen05 3xTF32 GEMM against L_kk^{-1} (default),
 *      0 = SIMT blocked substitution against 32x32 diagonal-block inverses
 *   4: CTAs of the lookahead panel-column FP32 update (0 = all SMs)
 *   5: SMs the bulk FP32 update yields to the panel kernels on request (default 0 =
 *      off on one GPU, where the panel chain is hidden; the P x Q path asks for 32)
 *   6: super-column width (owned tile columns) of the bulk FP32 update's output
 *      order, for L2 reuse of the panel operands (default 12; 0 = column-by-column
 *      slot order; single process row only)
 *   7, 8, 9: retired (round-1 single-CTA tcgen05 kernel A/B switches; -1)
 *  10: 1 = co-schedule the FP64 band update (programmatic dependent launch) on the
 *      SMs a capped bulk FP32 update leaves free (default), 0 = one after the other
 *  11: band update's SM share under option 10, in % of its work share (default 90)
 *  12: (round-1 RZ engine) 1 = bulk FP32 update on full-width 256 x 512 CTA-pair
 *      items (needs nb % 512 == 0; default), 0 = 256 x 256 items
 *  13: (round-1 RZ engine) 1 = the 256 x 512 update prefetches C rows into L2
 *  14: POTRF variant, all bitwise equal: 0 = one CTA (default); 1 = a cluster of
 *      nb/32 CTAs with the tile in distributed shared memory (0.35 vs 1.00 ms
 *      per 512-tile alone, but a 16-CTA cluster waits for a free GPC beside
 *      the co-scheduled bulk update); 2 = three small launches per 32-column
 *      block (no co-residency requirement)
 *  15: 1 = FP32 update on clusters of two CTA pairs sharing the B operand
 *  16: 1 = FP32 update diagnostics (mt_tcf_stats)
 *  17: 1 = the FP32 update applies C -= sum as a TMA reduce-add of -sum at L2
 *      (no C load round trip at the end of each item; bitwise equal; default),
 *      0 = C loaded into shared memory, C - sum stored */
int32_t mt_set_option(int32_t option, int32_t value);

/* Fill *theta from (variance, range, smoothness) on the host (covmath.py:72-95). */
int mt_matern_prepare(double variance, double spatial_range, double smoothness,
                      mt_matern* theta);

#ifdef __cplusplus
}
#endif
#endif /* MIXTILE_B200_H */
