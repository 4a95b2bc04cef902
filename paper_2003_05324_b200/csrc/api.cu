// C ABI + host-side scheduler of the tile Cholesky (replaces the reference's
// Python task graph and thread pool, factor.py:44-80,152-206,230-285).
//
// The right-looking DAG is issued as a stream/event schedule with lookahead 1:
//   panel stream (high priority):  upd(k -> column k+1), POTRF(k+1), TRSM(k+1)
//   caller stream:                 upd(k -> columns k+2 .. p-1)
// joined by two events per step, so the panel of step k+1 runs underneath the
// bulk update of step k.  Every tile still receives its updates in ascending
// k from exactly one kernel per step, so results equal the lookahead-0 order
// bit for bit (the reference's schedule invariance, factor.py:13-16).
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <functional>
#include <mutex>
#include <vector>

#include <cuda.h>

#include "mt_grid.cuh"

// kernels (other translation units)
int mt_generate_impl(const Grid& g, const double* locs, int metric, double radius,
                     const mt_matern& th, cudaStream_t st);
int mt_scan_duplicates_impl(const Grid& g, const double* locs, int metric, double radius,
                            cudaStream_t st);
int mt_matern_array_impl(const double* r, int64_t m, const mt_matern& th, double* out,
                         cudaStream_t st);
int mt_potrf_impl(const Grid& g, int k, int narrow, cudaStream_t st);
int mt_trsm_impl(const Grid& g, int k, cudaStream_t st,
                 const std::function<int()>* before = nullptr);
int mt_update_impl(const Grid& g, int k, int jlo, int jhi, cudaStream_t st);
int mt_logdet_impl(const Grid& g, double* out, double* work, cudaStream_t st);
int mt_solve_impl(const Grid& g, double* x, int64_t nrhs, int which, cudaStream_t st);
int mt_quad_impl(const Grid& g, const double* z, double* work, double* out, cudaStream_t st);
int mt_matvec_lower_impl(const Grid& g, const double* v, double* out, cudaStream_t st);
int mt_fwd_step_impl(const Grid& g, int i, double* x, cudaStream_t st, int which = 3);
int mt_trinv_impl(const Grid& g, int k, cudaStream_t st);
int mt_logdet_partials_impl(const Grid& g, double* partial, cudaStream_t st);
int mt_sumsq_impl(const double* x, int64_t m, double* work, double* out, cudaStream_t st);
int64_t mt_cross_work_doubles_impl(int64_t m, int64_t n);
int mt_cross_gemv_impl(const double* test, int64_t m, const double* train, int64_t n, int metric,
                       double radius, const mt_matern& th, const double* w, double* work,
                       double* out, cudaStream_t st);

// ------------------------------------------------------------------ errors
static thread_local char g_err[512] = "";

void mt_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int mt_cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return 0;
  mt_set_error("%s: %s", what, cudaGetErrorString(e));
  return 1;
}

#define CK(call, what) \
  do { if (mt_cuda_check((call), what)) return MT_E_CUDA; } while (0)
#define RC(call) \
  do { int rc__ = (call); if (rc__) return rc__; } while (0)

static int check_layout(const mt_tiles* g) {
  if (!g || g->n < 1 || g->nb < 1 || g->p != (int32_t)((g->n + g->nb - 1) / g->nb) ||
      g->t < 1 || g->t > g->p || g->mode < 0 || g->mode > 2 ||
      (g->mode == MT_MODE_DP && g->t != g->p) || !g->dp_pool || !g->status ||
      !g->scratch || (g->mode == MT_MODE_MP && g->t < g->p && !g->sp_pool) ||
      g->col_stride < 0 || g->row_stride < 0 ||
      ((g->col_stride > 1 || g->row_stride > 1) &&
       (g->col_offset < 0 || g->col_offset >= (g->col_stride > 0 ? g->col_stride : 1) ||
        g->row_offset < 0 || g->row_offset >= (g->row_stride > 0 ? g->row_stride : 1) ||
        !g->dpanel))) {
    mt_set_error("bad tile layout descriptor");
    return MT_E_BAD_ARG;
  }
  return MT_OK;
}
static int single_gpu_only(const mt_tiles* g, const char* what) {
  if (g->col_stride > 1 || g->row_stride > 1) {
    mt_set_error("%s operates on the full matrix; use the per-step multi-GPU entry points", what);
    return MT_E_BAD_ARG;
  }
  return MT_OK;
}

// ------------------------------------------------------ per-device context
namespace {
typedef CUresult (*WriteValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

struct DevCtx {
  cudaStream_t panel = nullptr;
  int* yield = nullptr;            // SM-yield request word of the bulk update
  WriteValueFn write_value = nullptr;
  std::vector<cudaEvent_t> ev;
  size_t next = 0;
  cudaEvent_t event() {
    cudaEvent_t e = ev[next];
    next = (next + 1) % ev.size();
    return e;
  }
};
std::mutex g_ctx_mu;
DevCtx* g_ctx[64] = {nullptr};

DevCtx* dev_ctx() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(g_ctx_mu);
  if (!g_ctx[dev]) {
    DevCtx* c = new DevCtx();
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&c->panel, cudaStreamNonBlocking, hi) != cudaSuccess) {
      delete c;
      return nullptr;
    }
    c->ev.resize(16);
    for (auto& e : c->ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess && cudaMalloc(&c->yield, 64) == cudaSuccess &&
        cudaMemset(c->yield, 0, 64) == cudaSuccess) {
      c->write_value = (WriteValueFn)fn;
    } else {
      c->yield = nullptr;
      cudaGetLastError();
    }
    g_ctx[dev] = c;
  }
  return g_ctx[dev];
}
}  // namespace

// ------------------------------------------------------------------ the DAG
// fwd (optional): a device vector (zero-padded, p*nb) on which the forward
// sweep y = L^{-1} x runs fused into the schedule: column k's step (the same
// TRSV + GEMV kernels as mt_solve's forward sweep, so results are identical)
// is issued right after panel k is final, underneath the bulk updates.
static int cholesky_schedule(const Grid& g, int lookahead, cudaStream_t main,
                             double* fwd = nullptr) {
  const int p = g.p;
  auto narrow_k = [&](int k) { return (g.mode == MT_MODE_MP && k + g.t <= p - 1) ? 1 : 0; };
  auto fwd_step = [&](int k, cudaStream_t s) { return fwd ? mt_fwd_step_impl(g, k, fwd, s) : MT_OK; };
  if (!lookahead || p < 3) {
    for (int k = 0; k < p; ++k) {
      RC(mt_potrf_impl(g, k, narrow_k(k), main));
      if (k + 1 < p) RC(mt_trsm_impl(g, k, main));
      RC(fwd_step(k, main));
      if (k + 1 < p) RC(mt_update_impl(g, k, k + 1, p, main));
    }
    return MT_OK;
  }
  DevCtx* ctx = dev_ctx();
  if (!ctx) { mt_set_error("cannot create the panel stream"); return MT_E_CUDA; }
  cudaStream_t pan = ctx->panel;
  // the bulk update (caller stream) yields SMs to the panel kernels on request
  Grid gb = g;
  const int ysms = mt_opt_yield_sms();
  const bool yield_on = ysms > 0 && ctx->yield && ctx->write_value;
  if (yield_on) gb.yield = ctx->yield;
  auto request = [&](unsigned v) -> int {
    if (!yield_on) return MT_OK;
    if (ctx->write_value((CUstream)pan, (CUdeviceptr)ctx->yield, v, 0) != CUDA_SUCCESS) {
      mt_set_error("cuStreamWriteValue32 failed");
      return MT_E_CUDA;
    }
    return MT_OK;
  };
  if (lookahead >= 2 && p >= 4) {
    if (g.nring < 3) {
      mt_set_error("lookahead 2 needs a layout with 3 panel slots (mt_tiles.panel_slots)");
      return MT_E_BAD_ARG;
    }
    // Lookahead depth 2: the panel stream keeps panels k+1 and k+2 ready while
    // the caller stream applies step k to columns k+3 ..; column j receives
    // steps j-2 and j-1 on the panel stream, the earlier ones from the bulk
    // updates.  Every tile still gets its updates in ascending k from the same
    // kernels, so the factor is bitwise identical to lookahead 0 / 1.
    std::vector<cudaEvent_t> panel_ev(p), step_ev(p);
    cudaEvent_t e0 = ctx->event();
    CK(cudaEventRecord(e0, main), "event record");
    CK(cudaStreamWaitEvent(pan, e0, 0), "stream wait");
    for (int j = 0; j < 2; ++j) {  // panels 0 and 1
      if (j == 1) RC(mt_update_impl(g, 0, 1, 2, pan));
      RC(mt_potrf_impl(g, j, narrow_k(j), pan));
      RC(mt_trsm_impl(g, j, pan));
      RC(fwd_step(j, pan));
      panel_ev[j] = ctx->event();
      CK(cudaEventRecord(panel_ev[j], pan), "event record");
    }
    for (int k = 0; k < p - 1; ++k) {
      const int j = k + 2;  // the panel the panel stream forms meanwhile
      if (j < p) {
        // column j got steps <= k-1 from the bulk updates; the ring slot of
        // panel j is panel k-1's, free once bulk(k-1) finished
        if (k >= 1) CK(cudaStreamWaitEvent(pan, step_ev[k - 1], 0), "stream wait");
        RC(mt_update_impl(g, k, j, j + 1, pan));
        RC(mt_update_impl(g, k + 1, j, j + 1, pan));
        RC(request(1u));
        RC(mt_potrf_impl(g, j, narrow_k(j), pan));
        if (j + 1 < p) {
          const std::function<int()> ask = [&]() { return request((unsigned)ysms); };
          RC(mt_trsm_impl(g, j, pan, yield_on ? &ask : nullptr));
        }
        RC(request(0u));
        RC(fwd_step(j, pan));
        panel_ev[j] = ctx->event();
        CK(cudaEventRecord(panel_ev[j], pan), "event record");
      }
      CK(cudaStreamWaitEvent(main, panel_ev[k], 0), "stream wait");
      if (k + 3 < p) RC(mt_update_impl(gb, k, k + 3, p, main));
      step_ev[k] = ctx->event();
      CK(cudaEventRecord(step_ev[k], main), "event record");
    }
    cudaEvent_t ef = ctx->event();
    CK(cudaEventRecord(ef, pan), "event record");
    CK(cudaStreamWaitEvent(main, ef, 0), "stream wait");
    return MT_OK;
  }
  cudaEvent_t e = ctx->event();
  CK(cudaEventRecord(e, main), "event record");
  CK(cudaStreamWaitEvent(pan, e, 0), "stream wait");
  RC(mt_potrf_impl(g, 0, narrow_k(0), pan));
  RC(mt_trsm_impl(g, 0, pan));
  RC(fwd_step(0, pan));
  for (int k = 0; k < p - 1; ++k) {
    cudaEvent_t ep = ctx->event();
    CK(cudaEventRecord(ep, pan), "event record");   // panel k ready
    CK(cudaStreamWaitEvent(main, ep, 0), "stream wait");
    // panel stream: column k+1 with panel k, then factor panel k+1; the
    // panel solves ask the bulk update for SMs (its CTAs exit between items)
    RC(mt_update_impl(g, k, k + 1, k + 2, pan));
    RC(request(1u));
    RC(mt_potrf_impl(g, k + 1, narrow_k(k + 1), pan));
    if (k + 2 < p) {
      const std::function<int()> ask = [&]() { return request((unsigned)ysms); };
      RC(mt_trsm_impl(g, k + 1, pan, yield_on ? &ask : nullptr));
    }
    // withdraw the request after every panel (also the last one, so the word
    // never carries into the next factorization or a later bulk update)
    RC(request(0u));
    RC(fwd_step(k + 1, pan));  // panel k+1 is final
    // caller stream: the rest of step k's trailing update
    RC(mt_update_impl(gb, k, k + 2, p, main));
    cudaEvent_t em = ctx->event();
    CK(cudaEventRecord(em, main), "event record");  // step k fully applied
    CK(cudaStreamWaitEvent(pan, em, 0), "stream wait");
  }
  cudaEvent_t ef = ctx->event();
  CK(cudaEventRecord(ef, pan), "event record");
  CK(cudaStreamWaitEvent(main, ef, 0), "stream wait");
  return MT_OK;
}

// ---------------------------------------------------------------- host math
namespace {
const double kLz[9] = {0.99999999999980993, 676.5203681218851,    -1259.1392167224028,
                       771.32342877765313,  -176.61502916214059,  12.507343278686905,
                       -0.13857109526572012, 9.9843695780195716e-6, 1.5056327351493116e-7};
double lanczos_gamma(double x) {  // covmath.py:40-49
  if (x < 0.5) return M_PI / (sin(M_PI * x) * lanczos_gamma(1.0 - x));
  x -= 1.0;
  double a = kLz[0];
  for (int i = 1; i < 9; ++i) a += kLz[i] / (x + i);
  double t = x + 7.0 + 0.5;
  return sqrt(2.0 * M_PI) * pow(t, x + 0.5) * exp(-t) * a;
}
double zeta_odd(int idx) {  // covmath.py:52-66 (sum k^-s, k < 60, + Euler-Maclaurin tail)
  const int s = 3 + 2 * idx, m = 60;
  double tot = 0.0;
  for (int k = 1; k < m; ++k) tot += pow((double)k, -s);
  tot += pow((double)m, 1 - s) / (s - 1);
  tot += 0.5 * pow((double)m, -s);
  tot += s * pow((double)m, -s - 1) / 12.0;
  tot -= s * (s + 1.0) * (s + 2.0) * pow((double)m, -s - 3) / 720.0;
  tot += s * (s + 1.0) * (s + 2.0) * (s + 3.0) * (s + 4.0) * pow((double)m, -s - 5) / 30240.0;
  return tot;
}
}  // namespace

// ------------------------------------------------------------ runtime options
static int g_engine = MT_ENGINE_TF32X3;
static int g_update_ctas = 0;  // 0 = all SMs
static int g_legacy_dmma = 0;  // 1 = register-staged DMMA band update (A/B comparisons)
static int g_pcol_ctas = 64;   // CTAs of the lookahead panel-column FP32 update (0 = all SMs)
static int g_yield_sms = 0;    // SMs the bulk update yields to the panel TRSM (0 = off: at g = 1 the panel chain is hidden, yielding cost 0.4%)
static int g_tc_trsm = 1;      // 1 = off-band TRSM as a tcgen05 3xTF32 GEMM against L_kk^{-1}
static int g_super_cols = 12;  // super-column width of the bulk FP32 update order (0 = slot order)
static int g_coschedule = 1;   // 1 = band DMMA update co-scheduled beside the capped FP32 update
static int g_cosched_pct = 90; // band update's SM share, % of its work share (option 11)
static int g_wide_items = 1;   // 1 = bulk FP32 update on 256 x 512 pair items (nb % 512 == 0)
static int g_wide_l2pf = 0;    // 1 = the 256 x 512 update stages each warp's C rows in L2
static int g_tcf_reduce = 1;    // 1 = tcf update applies C -= sum as a TMA reduce-add (no C load; default)
static int g_tcf_stats = 0;     // 1 = tcf kernels accumulate MMA-issuer wait cycles (diagnostics)
static int g_tcf_cluster4 = 0;  // 1 = RN tcgen05 update on 4-CTA clusters (B multicast across two pairs)
static int g_potrf_cluster = 0;  // 1 = POTRF on a cluster of nb/32 CTAs (tile in distributed smem; opt-in)
int mt_opt_engine() { return g_engine; }
int mt_opt_update_ctas() { return g_update_ctas; }
int mt_opt_legacy_dmma() { return g_legacy_dmma; }
int mt_opt_tc_trsm() { return g_tc_trsm; }
int mt_opt_pcol_ctas() { return g_pcol_ctas; }
int mt_opt_yield_sms() { return g_yield_sms; }
int mt_opt_super_cols() { return g_super_cols; }
int mt_opt_wide_items() { return g_wide_items; }
int mt_opt_wide_l2pf() { return g_wide_l2pf; }
int mt_opt_coschedule() { return g_coschedule; }
int mt_opt_coschedule_pct() { return g_cosched_pct; }
int mt_opt_potrf_cluster() { return g_potrf_cluster; }
int mt_opt_tcf_cluster4() { return g_tcf_cluster4; }
int mt_opt_tcf_stats() { return g_tcf_stats; }
int mt_opt_tcf_reduce() { return g_tcf_reduce; }

extern "C" {

int32_t mt_version(void) { return 11; }

/* option 0: FP32 update engine (0 FFMA SIMT, 1 tcgen05 3xTF32 round-to-nearest chunks,
 *           2 tcgen05 3xTF32 whole-K TMEM accumulation);
 * option 1: CTA cap of the bulk trailing update (0 = all SMs);
 * option 2: 1 = legacy register-staged DMMA band update;
 * option 3: 1 = off-band TRSM as a tcgen05 GEMM against L_kk^{-1} (default),
 *           0 = SIMT substitution against 32x32 inverses;
 * option 4: CTAs of the lookahead panel-column FP32 update (0 = all SMs);
 * option 5: SMs the bulk FP32 update yields to the panel TRSM (0 = off);
 * option 6: super-column width of the FP32 update's output order (default 8, 0 = slot order);
 * options 7-9: retired (round-1 single-CTA kernel A/B switches);
 * Returns the old value. */
int32_t mt_set_option(int32_t option, int32_t value) {
  int old = -1;
  if (option == 0) { old = g_engine; g_engine = value; }
  else if (option == 1) { old = g_update_ctas; g_update_ctas = value; }
  else if (option == 2) { old = g_legacy_dmma; g_legacy_dmma = value; }
  else if (option == 3) { old = g_tc_trsm; g_tc_trsm = value; }
  else if (option == 4) { old = g_pcol_ctas; g_pcol_ctas = value; }
  else if (option == 5) { old = g_yield_sms; g_yield_sms = value; }
  else if (option == 6) { old = g_super_cols; g_super_cols = value; }
  else if (option == 10) { old = g_coschedule; g_coschedule = value; }
  else if (option == 11) { old = g_cosched_pct; g_cosched_pct = value; }
  else if (option == 12) { old = g_wide_items; g_wide_items = value; }
  else if (option == 13) { old = g_wide_l2pf; g_wide_l2pf = value; }
  else if (option == 14) { old = g_potrf_cluster; g_potrf_cluster = value; }
  else if (option == 15) { old = g_tcf_cluster4; g_tcf_cluster4 = value; }
  else if (option == 16) { old = g_tcf_stats; g_tcf_stats = value; }
  else if (option == 17) { old = g_tcf_reduce; g_tcf_reduce = value; }
  return old;
}
const char* mt_last_error(void) { return g_err; }

int64_t mt_dp_tiles(int32_t p, int32_t t, int32_t mode) {
  if (mode == MT_MODE_DP) t = p;
  Grid g{};
  g.p = p; g.t = t; g.mode = mode;
  return g.bcol(p);
}
int64_t mt_sp_tiles(int32_t p, int32_t t, int32_t mode) {
  if (mode != MT_MODE_MP) return 0;
  Grid g{};
  g.p = p; g.t = t; g.mode = mode;
  return g.scol(p);
}

int64_t mt_scratch_tiles(int32_t p, int32_t t, int32_t mode, int32_t nb) {
  Grid g{};
  g.p = p; g.t = mode == MT_MODE_DP ? p : t; g.mode = mode; g.nb = nb;
  return 2 * g.slot_tiles();
}

int64_t mt_split_tiles(int32_t p, int32_t t, int32_t mode) {
  // 2 panels x p tiles x {hi, lo} + next-panel pre-split (p x {hi, lo}) + W = L^{-1} {hi, lo}
  return (mode == MT_MODE_MP && t < p) ? 6 * (int64_t)p + 2 : 0;
}

int mt_matern_prepare(double variance, double spatial_range, double smoothness, mt_matern* th) {
  if (!th || !(variance > 0) || !(spatial_range > 0) || !(smoothness > 0) || !isfinite(variance) ||
      !isfinite(spatial_range) || !isfinite(smoothness)) {
    mt_set_error("Matern parameters must be finite and > 0");
    return MT_E_BAD_ARG;
  }
  memset(th, 0, sizeof(*th));
  th->variance = variance;
  th->spatial_range = spatial_range;
  th->smoothness = smoothness;
  th->kind = smoothness == 0.5 ? 0 : (smoothness == 1.5 ? 1 : 2);
  th->nl = (int32_t)(smoothness + 0.5);
  const double mu = smoothness - th->nl;
  th->mu = mu;
  // Temme gammas (covmath.py:72-95)
  const double gp = 1.0 / lanczos_gamma(1.0 + mu);
  const double gm = 1.0 / lanczos_gamma(1.0 - mu);
  th->rp = gp;
  th->rm = gm;
  th->gam2 = 0.5 * (gm + gp);
  if (fabs(mu) >= 0.1) {
    th->gam1 = (gm - gp) / (2.0 * mu);
  } else if (mu == 0.0) {
    th->gam1 = -0.5772156649015329;
  } else {
    double acc = 0.5772156649015329, mu2 = mu * mu, mp = mu2;
    for (int idx = 0; idx < 10; ++idx) {
      acc += zeta_odd(idx) * mp / (3 + 2 * idx);
      mp *= mu2;
    }
    th->gam1 = gp * expm1(-2.0 * mu * acc) / (2.0 * mu);
  }
  th->fact = mu != 0.0 ? 1.0 / (sin(M_PI * mu) / (M_PI * mu)) : 1.0;  // 1/np.sinc(mu)
  th->scale = variance * pow(2.0, 1.0 - smoothness) / lanczos_gamma(smoothness);
  return MT_OK;
}

int mt_generate(const mt_tiles* t, const double* locs, int32_t metric, double radius,
                const mt_matern* theta, void* stream) {
  RC(check_layout(t));
  if (!locs || !theta) { mt_set_error("null locations/theta"); return MT_E_BAD_ARG; }
  return mt_generate_impl(make_grid(t), locs, metric, radius, *theta, (cudaStream_t)stream);
}

int mt_scan_duplicates(const mt_tiles* t, const double* locs, int32_t metric, double radius,
                       void* stream) {
  RC(check_layout(t));
  return mt_scan_duplicates_impl(make_grid(t), locs, metric, radius, (cudaStream_t)stream);
}

int mt_matern_array(const double* r, int64_t m, const mt_matern* theta, double* out,
                    void* stream) {
  if (!theta || (m > 0 && (!r || !out))) { mt_set_error("null argument"); return MT_E_BAD_ARG; }
  return mt_matern_array_impl(r, m, *theta, out, (cudaStream_t)stream);
}

int64_t mt_cross_work_doubles(int64_t m, int64_t n) { return mt_cross_work_doubles_impl(m, n); }

int mt_cross_gemv(const double* test, int64_t m, const double* train, int64_t n, int32_t metric,
                  double radius, const mt_matern* theta, const double* w, double* work,
                  double* out, void* stream) {
  if (m < 0 || n < 1 || !theta || (m > 0 && (!test || !train || !w || !work || !out)) ||
      (metric != MT_METRIC_EUCLIDEAN && metric != MT_METRIC_GREAT_CIRCLE)) {
    mt_set_error("mt_cross_gemv: bad arguments");
    return MT_E_BAD_ARG;
  }
  return mt_cross_gemv_impl(test, m, train, n, metric, radius, *theta, w, work, out,
                            (cudaStream_t)stream);
}

int mt_cholesky_quad(const mt_tiles* t, int32_t lookahead, const double* z, double* work,
                     double* out, void* stream) {
  RC(check_layout(t));
  RC(single_gpu_only(t, "mt_cholesky_quad"));
  if (!z || !work || !out) { mt_set_error("mt_cholesky_quad: null argument"); return MT_E_BAD_ARG; }
  const Grid g = make_grid(t);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t npad = (int64_t)g.p * g.nb;
  CK(cudaMemcpyAsync(work, z, npad * sizeof(double), cudaMemcpyDeviceToDevice, st), "quad copy");
  RC(cholesky_schedule(g, lookahead, st, work));
  return mt_sumsq_impl(work, npad, work + npad, out, st);
}

int mt_cholesky(const mt_tiles* t, int32_t lookahead, void* stream) {
  RC(check_layout(t));
  RC(single_gpu_only(t, "mt_cholesky"));
  return cholesky_schedule(make_grid(t), lookahead, (cudaStream_t)stream);
}

// ---- per-step entry points of the multi-GPU (2D block-cyclic) factorization
// POTRF(k) on the owner of tile (k, k); on a multi-GPU grid also the copy of
// L_kk into the FP64 panel ring (row k) and W = L_kk^{-1} for the tensor-core
// TRSM: what the column broadcast sends to the other ranks of process column k
int mt_panel_factor(const mt_tiles* t, int32_t k, void* stream) {
  RC(check_layout(t));
  const Grid g = make_grid(t);
  cudaStream_t st = (cudaStream_t)stream;
  if (k < 0 || k >= g.p || !g.owns(k, k)) {
    mt_set_error("mt_panel_factor: rank does not own tile (%d, %d)", k, k);
    return MT_E_BAD_ARG;
  }
  const int narrow = (g.mode == MT_MODE_MP && k + g.t <= g.p - 1) ? 1 : 0;
  RC(mt_potrf_impl(g, k, narrow, st));
  if (g.multi() && g.dpanel)
    CK(cudaMemcpyAsync(g.dpanel_tile(k, k), g.dtile(k, k), g.tile_elems() * sizeof(double),
                       cudaMemcpyDeviceToDevice, st), "L_kk to panel ring");
  if (g.multi() && g.mode == MT_MODE_MP && k + g.t < g.p && mt_tc_trsm_enabled(g))
    RC(mt_trinv_impl(g, k, st));
  return MT_OK;
}

// TRSM(k) of this rank's rows of tile column k (L_kk, its inverses and W present)
int mt_panel_solve(const mt_tiles* t, int32_t k, void* stream) {
  RC(check_layout(t));
  const Grid g = make_grid(t);
  if (k < 0 || k >= g.p || !g.owns_col(k)) {
    mt_set_error("mt_panel_solve: rank does not own tile column %d", k);
    return MT_E_BAD_ARG;
  }
  if (k + 1 < g.p) RC(mt_trsm_impl(g, k, (cudaStream_t)stream));
  return MT_OK;
}

// both, on a rank that owns tile (k, k) and the whole of column k (1 x Q grids)
int mt_panel(const mt_tiles* t, int32_t k, void* stream) {
  RC(check_layout(t));
  const Grid g = make_grid(t);
  if (k < 0 || k >= g.p || !g.owns_col(k) || g.rs > 1) {
    mt_set_error("mt_panel: rank does not own tile column %d", k);
    return MT_E_BAD_ARG;
  }
  RC(mt_panel_factor(t, k, stream));
  return mt_panel_solve(t, k, stream);
}

// element ranges of what the column broadcast of panel k carries on a P x Q
// grid (P > 1): {offset, count} of L_kk in dpanel (doubles), of the 32x32
// diagonal-block inverses in scratch (floats), of W's split in split (floats)
int mt_diag_regions(const mt_tiles* t, int32_t k, int64_t* out6) {
  RC(check_layout(t));
  const Grid g = make_grid(t);
  if (!out6 || k < 0 || k >= g.p) { mt_set_error("mt_diag_regions: bad arguments"); return MT_E_BAD_ARG; }
  const int64_t te = g.tile_elems();
  out6[0] = g.dpanel ? (g.dpanel_tile(k, k) - g.dpanel) : 0;
  out6[1] = g.dpanel ? te : 0;
  out6[2] = (float*)g.sinv64(k) - g.scratch;
  out6[3] = g.inv_tiles() * te;
  const bool w = g.split && g.mode == MT_MODE_MP && k + g.t < g.p;
  out6[4] = w ? g.winv_row() * g.nb : 0;
  out6[5] = w ? 2 * te : 0;
  return MT_OK;
}

int mt_update(const mt_tiles* t, int32_t k, int32_t jlo, int32_t jhi, void* stream) {
  RC(check_layout(t));
  const Grid g = make_grid(t);
  if (k < 0 || k >= g.p || jlo <= k || jhi > g.p) {
    mt_set_error("mt_update: bad step/column range");
    return MT_E_BAD_ARG;
  }
  return mt_update_impl(g, k, jlo, jhi, (cudaStream_t)stream);
}

int mt_update_ex(const mt_tiles* t, int32_t k, int32_t jlo, int32_t jhi, int32_t flags,
                 void* stream) {
  RC(check_layout(t));
  Grid g = make_grid(t);
  if (k < 0 || k >= g.p || jlo <= k || jhi > g.p) {
    mt_set_error("mt_update_ex: bad step/column range");
    return MT_E_BAD_ARG;
  }
  if (flags & 1) {
    DevCtx* ctx = dev_ctx();
    if (ctx && ctx->yield && ctx->write_value) g.yield = ctx->yield;
  }
  return mt_update_impl(g, k, jlo, jhi, (cudaStream_t)stream);
}

int mt_yield_request(int32_t sms, void* stream) {
  DevCtx* ctx = dev_ctx();
  if (!ctx || !ctx->yield || !ctx->write_value) return MT_OK;
  if (ctx->write_value((CUstream)stream, (CUdeviceptr)ctx->yield, (cuuint32_t)(sms > 0 ? sms : 0),
                       0) != CUDA_SUCCESS) {
    mt_set_error("cuStreamWriteValue32 failed");
    return MT_E_CUDA;
  }
  return MT_OK;
}

int mt_logdet_partials(const mt_tiles* t, double* partial, void* stream) {
  RC(check_layout(t));
  return mt_logdet_partials_impl(make_grid(t), partial, (cudaStream_t)stream);
}

int mt_fwd_step(const mt_tiles* t, int32_t i, double* x, void* stream) {
  RC(check_layout(t));
  return mt_fwd_step_impl(make_grid(t), i, x, (cudaStream_t)stream, 3);
}

int mt_fwd_step_ex(const mt_tiles* t, int32_t i, int32_t which, double* x, void* stream) {
  RC(check_layout(t));
  return mt_fwd_step_impl(make_grid(t), i, x, (cudaStream_t)stream, which);
}

int mt_sumsq(const double* x, int64_t m, double* work, double* out, void* stream) {
  if (!x || !work || !out || m < 0) { mt_set_error("mt_sumsq: bad arguments"); return MT_E_BAD_ARG; }
  return mt_sumsq_impl(x, m, work, out, (cudaStream_t)stream);
}

int mt_local_tiles(int32_t p, int32_t t_, int32_t mode, int32_t col_stride, int32_t col_offset,
                   int64_t* ndp, int64_t* nsp) {
  Grid g{};
  g.p = p; g.t = mode == MT_MODE_DP ? p : t_; g.mode = mode;
  g.cs = col_stride > 0 ? col_stride : 1; g.c0 = col_offset;
  if (ndp) *ndp = g.nband();
  if (nsp) *nsp = g.noff();
  return MT_OK;
}

int64_t mt_dpanel_tiles(int32_t p, int32_t t_, int32_t mode) {
  (void)t_; (void)mode;
  return mt_dpanel_tiles_ex(p, 1, 2);
}

int mt_local_tiles_ex(int32_t p, int32_t t_, int32_t mode, int32_t row_stride, int32_t row_offset,
                      int32_t col_stride, int32_t col_offset, int64_t* ndp, int64_t* nsp) {
  Grid g{};
  g.p = p; g.t = mode == MT_MODE_DP ? p : t_; g.mode = mode;
  g.cs = col_stride > 0 ? col_stride : 1; g.c0 = col_offset;
  g.rs = row_stride > 0 ? row_stride : 1; g.r0 = row_offset;
  if (ndp) *ndp = g.nband();
  if (nsp) *nsp = g.noff();
  return MT_OK;
}

// both panel rings hold every tile row (ring order): 2 panels x pring tiles
int64_t mt_dpanel_tiles_ex(int32_t p, int32_t row_stride, int32_t col_stride) {
  Grid g{};
  g.p = p;
  g.rs = row_stride > 0 ? row_stride : 1;
  g.cs = col_stride > 0 ? col_stride : 1;
  return 2 * (int64_t)g.pring();
}

int64_t mt_split_tiles_ex(int32_t p, int32_t t_, int32_t mode, int32_t row_stride,
                          int32_t col_stride) {
  if (!(mode == MT_MODE_MP && t_ < p)) return 0;
  Grid g{};
  g.p = p;
  g.rs = row_stride > 0 ? row_stride : 1;
  g.cs = col_stride > 0 ? col_stride : 1;
  return 4 * (int64_t)g.pring() + 2 * (int64_t)p + 2;
}

int mt_ring_tiles(int32_t p, int32_t t_, int32_t mode, int32_t nb, int32_t row_stride,
                  int32_t col_stride, int32_t slots, int64_t* scratch, int64_t* split,
                  int64_t* dpanel) {
  Grid g{};
  g.p = p; g.t = mode == MT_MODE_DP ? p : t_; g.mode = mode; g.nb = nb;
  g.rs = row_stride > 0 ? row_stride : 1;
  g.cs = col_stride > 0 ? col_stride : 1;
  g.nring = slots > 2 ? slots : 2;
  if (scratch) *scratch = (int64_t)g.nring * g.slot_tiles();
  if (split) *split = (mode == MT_MODE_MP && g.t < p) ? g.split_rows() / nb : 0;
  if (dpanel) *dpanel = (int64_t)g.nring * g.pring();
  return MT_OK;
}

int32_t mt_ring_pos(int32_t p, int32_t row_stride, int32_t col_stride, int32_t i) {
  Grid g{};
  g.p = p;
  g.rs = row_stride > 0 ? row_stride : 1;
  g.cs = col_stride > 0 ? col_stride : 1;
  return g.ring_pos(i);
}

int64_t mt_work_doubles(const mt_tiles* t) {
  return (int64_t)t->p * t->nb + 2048 + t->p;
}

int mt_logdet(const mt_tiles* t, double* work, double* out, void* stream) {
  RC(check_layout(t));
  RC(single_gpu_only(t, "mt_logdet"));
  return mt_logdet_impl(make_grid(t), out, work, (cudaStream_t)stream);
}

int mt_solve(const mt_tiles* t, double* x, int64_t nrhs, int32_t which, void* stream) {
  RC(check_layout(t));
  RC(single_gpu_only(t, "mt_solve"));
  if (nrhs < 1 || which < 1 || which > 3) { mt_set_error("bad solve arguments"); return MT_E_BAD_ARG; }
  return mt_solve_impl(make_grid(t), x, nrhs, which, (cudaStream_t)stream);
}

int mt_quad(const mt_tiles* t, const double* z, double* work, double* out, void* stream) {
  RC(check_layout(t));
  RC(single_gpu_only(t, "mt_quad"));
  return mt_quad_impl(make_grid(t), z, work, out, (cudaStream_t)stream);
}

int mt_matvec_lower(const mt_tiles* t, const double* v, double* out, void* stream) {
  RC(check_layout(t));
  RC(single_gpu_only(t, "mt_matvec_lower"));
  return mt_matvec_lower_impl(make_grid(t), v, out, (cudaStream_t)stream);
}

int mt_reset_status(const mt_tiles* t, void* stream) {
  RC(check_layout(t));
  const int64_t init[4] = {-1, 0, 0, 0};
  CK(cudaMemcpyAsync(t->status, init, sizeof(init), cudaMemcpyHostToDevice, (cudaStream_t)stream),
     "status reset");
  // the host array is on the stack: make the copy complete before returning
  CK(cudaStreamSynchronize((cudaStream_t)stream), "status reset sync");
  return MT_OK;
}

int mt_evaluate(const mt_tiles* t, const double* locs, int32_t metric, double radius,
                const mt_matern* theta, const double* z, double* work, double* out2,
                int32_t lookahead, void* stream) {
  RC(check_layout(t));
  RC(single_gpu_only(t, "mt_evaluate"));
  const Grid g = make_grid(t);
  cudaStream_t st = (cudaStream_t)stream;
  RC(mt_generate_impl(g, locs, metric, radius, *theta, st));
  // quad = ||L^{-1} z||^2 with the forward sweep fused into the factorization
  const int64_t npad = (int64_t)g.p * g.nb;
  CK(cudaMemcpyAsync(work, z, npad * sizeof(double), cudaMemcpyDeviceToDevice, st), "quad copy");
  RC(cholesky_schedule(g, lookahead, st, work));
  RC(mt_logdet_impl(g, out2, work + npad + 2048, st));
  RC(mt_sumsq_impl(work, npad, work + npad, out2 + 1, st));
  return MT_OK;
}

int mt_read_status(const mt_tiles* t, int64_t* bad_pivot, int64_t* overflow, int64_t* dups,
                   void* stream) {
  RC(check_layout(t));
  int64_t h[4];
  CK(cudaMemcpyAsync(h, t->status, sizeof(h), cudaMemcpyDeviceToHost, (cudaStream_t)stream),
     "status read");
  CK(cudaStreamSynchronize((cudaStream_t)stream), "status sync");
  if (bad_pivot) *bad_pivot = h[0];
  if (overflow) *overflow = h[1];
  if (dups) *dups = h[2];
  if (h[1] > 0) { mt_set_error("%lld value(s) exceed FP32 range during narrowing", (long long)h[1]); return MT_E_OVERFLOW; }
  if (h[0] >= 0) { mt_set_error("matrix not positive definite at global pivot %lld", (long long)h[0]); return MT_E_NOT_SPD; }
  return MT_OK;
}

// host tile transfer: host buffer is (rows_i x rows_j) column-major
static int tile_xfer(const mt_tiles* t, int32_t i, int32_t j, int32_t which, void* host, bool get,
                     cudaStream_t st) {
  RC(check_layout(t));
  const Grid g = make_grid(t);
  if (i < 0 || j < 0 || i >= g.p || j > i || !g.present(i, j) || (which == 0) != g.band(i, j) ||
      !g.owns(i, j)) {
    mt_set_error("tile (%d,%d) not stored in the requested pool", i, j);
    return MT_E_BAD_ARG;
  }
  const int nb = g.nb, ri = g.rows(i), rj = g.rows(j);
  const size_t es = which == 0 ? 8 : 4;
  void* dev = which == 0 ? (void*)g.dtile(i, j) : (void*)g.stile(i, j);
  std::vector<unsigned char> buf((size_t)nb * nb * es);
  if (get) {
    CK(cudaMemcpyAsync(buf.data(), dev, buf.size(), cudaMemcpyDeviceToHost, st), "tile get");
    CK(cudaStreamSynchronize(st), "tile get sync");
    for (int r = 0; r < ri; ++r)
      for (int c = 0; c < rj; ++c)
        memcpy((unsigned char*)host + ((size_t)c * ri + r) * es, &buf[((size_t)r * nb + c) * es], es);
  } else {
    memset(buf.data(), 0, buf.size());
    for (int r = 0; r < nb; ++r)
      for (int c = 0; c < nb; ++c) {
        unsigned char* d = &buf[((size_t)r * nb + c) * es];
        if (r < ri && c < rj) {
          memcpy(d, (const unsigned char*)host + ((size_t)c * ri + r) * es, es);
        } else if (i == j && r == c) {  // padded diagonal -> identity
          if (es == 8) { double one = 1.0; memcpy(d, &one, 8); }
          else { float one = 1.0f; memcpy(d, &one, 4); }
        }
      }
    CK(cudaMemcpyAsync(dev, buf.data(), buf.size(), cudaMemcpyHostToDevice, st), "tile put");
    CK(cudaStreamSynchronize(st), "tile put sync");
  }
  return MT_OK;
}

int mt_get_tile(const mt_tiles* t, int32_t i, int32_t j, int32_t which, void* host, void* stream) {
  return tile_xfer(t, i, j, which, host, true, (cudaStream_t)stream);
}
int mt_put_tile(const mt_tiles* t, int32_t i, int32_t j, int32_t which, const void* host,
                void* stream) {
  return tile_xfer(t, i, j, which, (void*)host, false, (cudaStream_t)stream);
}

int mt_evaluate_host(int64_t n, int32_t nb, int32_t mode, int32_t t_, const double* locs,
                     const double* z, int32_t metric, double radius, const mt_matern* theta,
                     double* out2, int64_t* bad_pivot) {
  if (n < 1 || nb < 1 || !locs || !z || !theta || !out2) { mt_set_error("bad arguments"); return MT_E_BAD_ARG; }
  mt_tiles t{};
  t.n = n; t.nb = nb; t.p = (int32_t)((n + nb - 1) / nb);
  t.mode = mode; t.t = mode == MT_MODE_DP ? t.p : t_;
  if (t.t < 1 || t.t > t.p) { mt_set_error("diag_thick out of range"); return MT_E_BAD_ARG; }
  const int64_t te = (int64_t)nb * nb, npad = (int64_t)t.p * nb;
  const size_t b_dp = mt_dp_tiles(t.p, t.t, mode) * te * 8, b_sp = mt_sp_tiles(t.p, t.t, mode) * te * 4,
               b_sc = mt_scratch_tiles(t.p, t.t, mode, nb) * te * 4;
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
  double *d_locs = nullptr, *d_z = nullptr, *d_work = nullptr, *d_out = nullptr;
  int rc = MT_OK;
  auto al = [&](void** p, size_t b) { return mt_cuda_check(cudaMallocAsync(p, b ? b : 16, st), "alloc"); };
  if (al((void**)&t.dp_pool, b_dp) || al((void**)&t.sp_pool, b_sp) || al((void**)&t.scratch, b_sc) ||
      al((void**)&t.status, 32) || al((void**)&d_locs, npad * 16) || al((void**)&d_z, npad * 8) ||
      al((void**)&d_work, mt_work_doubles(&t) * 8) || al((void**)&d_out, 16)) {
    rc = MT_E_CUDA;
  }
  // the tensor-core engine's split buffer, as TileMatrix allocates it
  // (tilestore.py): the C entry point runs the same kernels as the Python path
  const int64_t nsplit = (mode == MT_MODE_MP && nb % 256 == 0) ? mt_split_tiles(t.p, t.t, mode) : 0;
  if (!rc && nsplit > 0 && al((void**)&t.split, (size_t)nsplit * te * 4)) rc = MT_E_CUDA;
  if (!rc) {
    const int64_t init[4] = {-1, 0, 0, 0};
    cudaMemcpyAsync(t.status, init, sizeof(init), cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(d_z, 0, npad * 8, st);
    cudaMemcpyAsync(d_locs, locs, n * 16, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_z, z, n * 8, cudaMemcpyHostToDevice, st);
    rc = mt_evaluate(&t, d_locs, metric, radius, theta, d_z, d_work, d_out, 1, st);
    if (!rc) {
      double h[2];
      cudaMemcpyAsync(h, d_out, 16, cudaMemcpyDeviceToHost, st);
      int64_t bp = -1;
      rc = mt_read_status(&t, &bp, nullptr, nullptr, st);
      if (bad_pivot) *bad_pivot = bp;
      out2[0] = h[0];
      out2[1] = h[1];
    }
  }
  cudaFreeAsync(t.dp_pool, st); cudaFreeAsync(t.sp_pool, st); cudaFreeAsync(t.scratch, st);
  cudaFreeAsync(t.status, st); cudaFreeAsync(d_locs, st); cudaFreeAsync(d_z, st);
  if (t.split) cudaFreeAsync(t.split, st);
  cudaFreeAsync(d_work, st); cudaFreeAsync(d_out, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  return rc;
}

}  // extern "C"
