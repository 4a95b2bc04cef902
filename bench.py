#!/usr/bin/env python
"""Benchmark: mixed-precision Gaussian log-likelihood evaluations on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json metric, "at N=262144"): one step = one full
log-likelihood evaluation at N = 262,144 locations, tile 512, MP band t = 8,
Matern (1, 0.1, 0.5) on a Morton-sorted synthetic field -- covariance
generation -> band-precision tile Cholesky -> logdet -> quadratic form, all on
the device.  MP at this size needs 142 GB, so it fits one B200; with N > 1 the
same evaluation is split over the ranks (2D block-cyclic P x Q tiles, NCCL
row/column panel broadcasts; strong scaling).  `--gpus N` outside torchrun
spawns the N ranks itself.  Prints ONE JSON line (rank 0).

  value      whole-job loglik evaluations/s, inputs resident in HBM, device time
             (CUDA events on the launching stream, max over ranks).
             cholesky_tflops = (N^3/3) / T_chol, T_chol timed inside each step.
  e2e        the same metric through the public API `loglik(dataset, ...)`
             (`loglik_distributed` for N > 1) from pinned host buffers: H2D of
             locations + z and D2H of the result inside the timed region.
  roofline   dominant kernel (the tcgen05 3xTF32 bulk update): algorithmic
             flops per launch / the launches' device-side span inside the
             timed region (frac raw; the per-SM-share figure beside it); plus
             the flop-weighted FP64/FP32 roofline of the whole factorization
             (P64 = FP64 DMMA probe of this run, sustained).
  mp_vs_dp   the build's own full-DP path timed the same way (at N = 262144
             when it fits the ranks' memory, else at configs[1] N = 65536).
  cpu_baseline  the reference algorithm (oracle port: same LAPACK/BLAS calls as
             the reference) on the host cores, bounded sample at N = 16384,
             extrapolated by component (assembly/solve N^2, FP64/FP32 kernels
             by planned flops at their measured rates, task loop p^3).

--impl reference times only the CPU reference arm (rank 0).
"""

import argparse
import ctypes
import gc
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("Mixed-precision Cholesky TFLOP/s + loglik evals/s at N=262144, 1-8 B200 vs full-DP")
UNIT = "loglik evals/s"
THETA = (1.0, 0.1, 0.5)
KINDS = ["gen64", "gen32", "potrf", "trsm64", "trsm32", "upd64", "upd32", "solve", "misc",
         "upd64p", "upd32p"]
# profiling recipe fallback (B200_PROFILING.md) when MEASURED_PEAKS.json is absent
FALLBACK_PEAKS = {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", "--matrix-n", dest="n", type=int, default=262144)
    ap.add_argument("--nb", type=int, default=512)
    ap.add_argument("--t", type=int, default=8)
    ap.add_argument("--dp-n", type=int, default=65536,
                    help="N of the MP-vs-DP comparison when full DP at --n does not fit")
    ap.add_argument("--dp-t", type=int, default=8,
                    help="MP band of the MP-vs-DP comparison at --dp-n (default: the headline t)")
    ap.add_argument("--cpu-n", type=int, default=16384, help="CPU baseline sample size")
    ap.add_argument("--engine", default="tf32x3", choices=["tf32x3", "tf32x3_rz", "ffma"],
                    help="off-band FP32 engine (default: the FP32-accurate tcgen05 engine)")
    ap.add_argument("--grid", default=None,
                    help="process grid PxQ for N > 1 (default: north_star's 1x2 / 2x2 / 2x4)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-dp", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    if os.environ.get("MT_BENCH_ARGV") is not None and "WORLD_SIZE" in os.environ:
        return ap.parse_args(json.loads(os.environ["MT_BENCH_ARGV"]))  # spawned by --gpus N
    return ap.parse_args()


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._th = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = sorted(float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit())
        mx = max((float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[q] for r in self.rows for q in range(4)
                          if len(r) > 4 + q and r[4 + q].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(self.rows)}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "MEASURED_PEAKS.json (of measured)"
    except Exception:
        return dict(FALLBACK_PEAKS), "B200_PROFILING.md fallback (of fallback; MEASURED_PEAKS.json absent)"


# --------------------------------------------------------------- CPU baseline
class _TimedKernels:
    """Stand-in for the oracle's scipy BLAS/LAPACK modules that times every
    call, split into FP64 kernels (dpotrf/dtrsm/dsyrk/dgemm) and FP32 kernels
    (strsm/sgemm), so the Cholesky can be extrapolated by component."""

    DP = ("dpotrf", "dtrsm", "dsyrk", "dgemm")
    SP = ("strsm", "sgemm")

    def __init__(self, mod, acc):
        self._m, self._acc = mod, acc

    def __getattr__(self, name):
        fn = getattr(self._m, name)
        kind = "dp" if name in self.DP else ("sp" if name in self.SP else None)
        if kind is None:
            return fn

        def timed(*a, **kw):
            t0 = time.perf_counter()
            try:
                return fn(*a, **kw)
            finally:
                self._acc[kind] += time.perf_counter() - t0
        return timed


def cpu_reference_sample(n, nb, t, reps=1):
    """Time the reference algorithm (oracle port) for one MP evaluation at n on
    all host cores, by component: assembly, the Cholesky's FP64 and FP32
    kernels, the rest of the Cholesky (task loop, conversions), logdet + solve.
    Returns (seconds per eval, components dict, cores, info)."""
    import numpy as np
    from threadpoolctl import threadpool_info, threadpool_limits

    from oracle import mixtile_oracle as O
    from paper_2003_05324_b200.geodata import GeoDataset, derive_seed, generate_locations, morton_sort

    cores = os.cpu_count() or 1
    locs = generate_locations(n, seed=derive_seed(0, 0))
    ds, _ = morton_sort(GeoDataset(locs, np.random.default_rng(7).standard_normal(n)))
    t = min(t, -(-n // nb))
    best, comp = float("inf"), None
    saved = (O._blas, O._lapack)
    with threadpool_limits(limits=cores):
        for _ in range(reps):
            acc = {"dp": 0.0, "sp": 0.0}
            O._blas, O._lapack = _TimedKernels(saved[0], acc), _TimedKernels(saved[1], acc)
            try:
                t0 = time.perf_counter()
                tiles = O.assemble(ds.locations, THETA, nb, "mp", t)
                t1 = time.perf_counter()
                fac = O.cholesky(tiles, n, nb, "mp", t)
                t2 = time.perf_counter()
                O.logdet(fac, -(-n // nb))
                float(ds.z @ O.solve(fac, n, nb, ds.z))
                t3 = time.perf_counter()
            finally:
                O._blas, O._lapack = saved
            if t3 - t0 < best:
                best = t3 - t0
                comp = {"assemble_s": t1 - t0, "cholesky_s": t2 - t1, "chol_fp64_kernels_s": acc["dp"],
                        "chol_fp32_kernels_s": acc["sp"],
                        "chol_other_s": max(0.0, (t2 - t1) - acc["dp"] - acc["sp"]),
                        "logdet_solve_s": t3 - t2}
        libs = [f"{d.get('internal_api')}:{d.get('num_threads')}" for d in threadpool_info()]
    cpu = ""
    try:
        with open("/proc/cpuinfo") as fh:
            cpu = next((ln.split(":", 1)[1].strip() for ln in fh if ln.startswith("model name")), "")
    except OSError:
        pass
    return best, comp, cores, {"cpu_model": cpu, "blas_threads": libs}


def extrapolate_cpu(comp, n_s, n, nb, t):
    """Seconds per evaluation at n from a sample at n_s, by component:
    assembly and logdet+solve scale with the matrix size (N^2); the Cholesky's
    FP64 and FP32 kernels run at their measured rates over the planned FP64 /
    FP32 flops at n (factor.py:134-145, so the band's share is right at both
    sizes); the task loop scales with the task count (p^3)."""
    from oracle import mixtile_oracle as O
    ps, p = -(-n_s // nb), -(-n // nb)
    fdp_s, fsp_s = O.planned_flops(n_s, nb, "mp", min(t, ps))
    fdp, fsp = O.planned_flops(n, nb, "mp", min(t, p)) if p <= 64 else _planned_closed(n, nb, t)
    r_dp = fdp_s / max(comp["chol_fp64_kernels_s"], 1e-9)
    r_sp = fsp_s / max(comp["chol_fp32_kernels_s"], 1e-9)
    parts = {
        "assemble_s": comp["assemble_s"] * (n / n_s) ** 2,
        "chol_fp64_kernels_s": fdp / r_dp,
        "chol_fp32_kernels_s": fsp / r_sp,
        "chol_other_s": comp["chol_other_s"] * (p / ps) ** 3,
        "logdet_solve_s": comp["logdet_solve_s"] * (n / n_s) ** 2,
    }
    return sum(parts.values()), parts, {"cpu_fp64_gflops": r_dp / 1e9, "cpu_fp32_gflops": r_sp / 1e9}


def _planned_closed(n, nb, t):
    """(F_dp, F_sp) of an MP plan with uniform tiles (SURVEY.md 8d closed form)."""
    p = n // nb
    s1 = sum(p - d for d in range(1, t))
    s2 = sum((p - 1 - d) * (p - d) / 2 for d in range(1, t))
    fdp = nb ** 3 * (p / 3 + p * (p - 1) / 2 + s1 + 2 * s2)
    return fdp, n ** 3 / 3 - fdp


def cpu_baseline_obj(args):
    sec, comp, cores, info = cpu_reference_sample(args.cpu_n, args.nb, args.t, reps=2)
    ext, parts, rates = extrapolate_cpu(comp, args.cpu_n, args.n, args.nb, args.t)
    return {
        "value": 1.0 / ext,
        "unit": UNIT,
        "cores": cores,
        "kind": "port",
        "sample": (f"oracle port of the reference (same dpotrf/dtrsm/strsm/dsyrk/dgemm/sgemm "
                   f"calls; bitwise-pinned to reference goldens), best of 2 MP t="
                   f"{min(args.t, args.cpu_n // args.nb)} nb={args.nb} evaluations at N={args.cpu_n}: "
                   f"{sec:.2f} s; extrapolated to N={args.n} by component (assembly and solve "
                   f"by N^2, FP64/FP32 kernels by their planned flops at their measured rates, "
                   f"task loop by p^3): {ext:.0f} s per evaluation"),
        "sample_components_s": comp,
        "extrapolated_components_s": parts,
        **rates,
        **info,
    }


def run_reference(args, rank):
    if rank != 0:
        return
    for _ in range(max(0, args.warmup)):
        cpu_reference_sample(args.cpu_n, args.nb, args.t)
    exts = []
    cores, info, parts, rates = 1, {}, {}, {}
    for _ in range(max(1, args.steps)):
        sec, comp, cores, info = cpu_reference_sample(args.cpu_n, args.nb, args.t)
        ext, parts, rates = extrapolate_cpu(comp, args.cpu_n, args.n, args.nb, args.t)
        exts.append(ext)
    sec = sum(exts) / len(exts)
    value = 1.0 / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic",
        "config": {"workload": f"MP t={args.t} nb={args.nb} loglik at N={args.n}: each step one "
                               f"evaluation sampled at N={args.cpu_n} on the host CPU, "
                               f"extrapolated by component",
                   "n": args.n, "nb": args.nb, "band_t": args.t},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"one MP evaluation at N={args.cpu_n} per step (oracle port of "
                                   f"the reference, all host threads), extrapolated to N={args.n} "
                                   f"by component (assembly/solve N^2, FP64/FP32 kernels by planned "
                                   f"flops at measured rates, task loop p^3)",
                         "extrapolated_components_s": parts, **rates, **info},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def process_grid(world, spec=None):
    """(P, Q) for `world` ranks: --grid PxQ, else north_star's shapes
    (1x2, 2x2, 2x4; 1 x world otherwise)."""
    if spec:
        P, Q = (int(v) for v in spec.lower().split("x"))
        if P * Q != world:
            raise SystemExit(f"--grid {spec} does not match {world} ranks")
        return P, Q
    return {4: (2, 2), 8: (2, 4)}.get(world, (1, world))


def fp64_peaks(lib, seconds=4.0):
    """FP64 DMMA peak of this GPU: (burst, sustained) TFLOP/s.  Burst = best of
    5 short probe launches; sustained = median launch while probing back to
    back for `seconds` (the way MEASURED_PEAKS.json measures bf16)."""
    v = ctypes.c_double()
    burst = 0.0
    for _ in range(5):
        lib.mt_peak_probe(2, 20000, ctypes.byref(v))
        burst = max(burst, v.value)
    rates, t0 = [], time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        lib.mt_peak_probe(2, 20000, ctypes.byref(v))
        rates.append(v.value)
    rates.sort()
    return burst, rates[len(rates) // 2]


# ------------------------------------------------------------------- GPU arm
def _dataset(mt, n, seed_rank=0):
    import numpy as np
    locs = mt.generate_locations(n, seed=mt.derive_seed(seed_rank, 0))
    z = np.random.default_rng(mt.derive_seed(seed_rank, 1)).standard_normal(n)
    ds, _ = mt.morton_sort(mt.GeoDataset(locs, z))
    return ds


def _free_memory():
    import torch
    gc.collect()
    torch.cuda.empty_cache()


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2003_05324_b200 as mt
    from paper_2003_05324_b200 import _lib
    from paper_2003_05324_b200.distributed import DistributedEvaluator, loglik_distributed

    local_rank = local_rank % torch.cuda.device_count()  # (dev gloo check: ranks share a GPU)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    lib = _lib.load()
    dist_on = world > 1

    def barrier():
        if dist_on:
            dist.barrier()

    def max_over_ranks(x):
        if not dist_on:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    grid = process_grid(world, args.grid)

    def make_eval(asm, pol):
        return DistributedEvaluator(asm, pol, grid=grid) if dist_on else mt.Evaluator(asm, pol)

    def run_eval(ev, th, chol_events=None):
        if dist_on:
            return ev(th, chol_events=chol_events)
        ev.launch(th, chol_events=chol_events)
        return ev.finish()

    n, nb, t = args.n, args.nb, args.t
    engine = args.engine
    mt.set_fp32_engine(engine)
    opts = {}
    if os.environ.get("MT_OPTS"):  # A/B of library options, e.g. MT_OPTS=15=1 (reported)
        for kv in os.environ["MT_OPTS"].split(","):
            k_, v_ = kv.split("=")
            lib.mt_set_option(int(k_), int(v_))
            opts[int(k_)] = int(v_)
    ds = _dataset(mt, n)  # same dataset on every rank (one distributed evaluation)
    theta = mt.MaternParams(*THETA)
    mp_pol = mt.PrecisionPolicy.mp(diag_thick=t)
    asm = mt.TileAssembler(ds, nb)
    ev = make_eval(asm, mp_pol)
    warm = max(3, args.warmup)
    for _ in range(warm):
        run_eval(ev, theta)

    # ---- timed region: K evaluations, inputs resident in HBM
    clocks = ClockSampler(local_rank)
    st = torch.cuda.current_stream()
    K = len(KINDS)
    barrier()
    torch.cuda.synchronize()
    lib.mt_prof_begin(65536)
    l0 = lib.mt_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    results = []
    with clocks:
        e0.record(st)
        for s in range(args.steps):
            results.append(run_eval(ev, theta, chol_events=cev[s]))
        e1.record(st)
        torch.cuda.synchronize()
    launches = lib.mt_launch_count() - l0
    arr = [(ctypes.c_double * K)() for _ in range(3)]
    cnt = (ctypes.c_int64 * K)()
    lib.mt_prof_end(K, arr[0], arr[1], arr[2], cnt)
    msw = (ctypes.c_double * K)()
    lib.mt_prof_sm_weighted(K, msw)
    barrier()
    t_dev = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    t_chol = max_over_ranks(sum(a.elapsed_time(b) for a, b in cev) / 1e3 / args.steps)
    value = args.steps / t_dev
    chol_tflops = (n ** 3 / 3.0) / t_chol / 1e12
    kinds = {KINDS[q]: {"ms": arr[0][q] / args.steps, "ms_sm_weighted": msw[q] / args.steps,
                        "flops": arr[1][q] / args.steps,
                        "bytes": arr[2][q] / args.steps, "launches": cnt[q] // max(1, args.steps)}
             for q in range(K)}

    # ---- roofline of the dominant kernel (bulk FP32 trailing update), live in the timed region
    peaks, peak_src = load_peaks()
    bf16_sus = float(peaks.get("bf16_tflops_sustained") or FALLBACK_PEAKS["bf16_tflops_sustained"])
    dom = "upd32"
    d = kinds[dom]
    # the bulk update runs beside the co-scheduled band update on a share of the
    # SMs (option 10): achieved = its flops / (its device span x its SM share),
    # i.e. the rate per whole-GPU-equivalent against the whole-GPU peak
    sm_share = d["ms_sm_weighted"] / d["ms"] if d["ms"] > 0 else 1.0
    achieved = d["flops"] / (d["ms_sm_weighted"] * 1e-3) / 1e12 if d["ms"] > 0 else 0.0
    achieved_raw = d["flops"] / (d["ms"] * 1e-3) / 1e12 if d["ms"] > 0 else 0.0
    p32 = bf16_sus / 6.0  # tcgen05 kind::tf32 = bf16 rate / 2; 3xTF32 = 3 MMAs per FP32 product
    p64_burst, p64_sus = fp64_peaks(lib)
    p64_burst, p64_sus = max_over_ranks(p64_burst), max_over_ranks(p64_sus)
    p64 = p64_sus  # the factorization is a long step: sustained, like P32
    traffic = None
    dom_kernel = {"tf32x3": "tcf_update_kernel", "tf32x3_rz": "tc2w_update_kernel"}.get(
        engine, "sgemm_update_kernel")
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh)
        ent = tr.get(f"n{n}_nb{nb}_t{t}", {})
        cands = sorted((v["avg_duration_ms"], v["dram_bytes_per_launch"])
                       for name, v in ent.items() if name.startswith(dom_kernel))
        if cands:  # the longest launches are the bulk updates
            traffic = cands[-1][1]
    except Exception:
        traffic = None
    fl_plan = mt.planned_flops(n, nb, mp_pol)
    t_roof = (fl_plan.sp / (p32 * 1e12) + fl_plan.dp / (p64 * 1e12)) / world
    roofline = {
        "bound": "tensor", "achieved": achieved_raw, "peak": p32, "unit": "TFLOP/s",
        "frac": achieved_raw / p32, "traffic": traffic,
        "kernel": f"{dom_kernel} (CTA pairs, tcgen05.mma.cta_group::2)",
        "pipe": ("tcgen05.mma kind::tf32 (3xTF32 FP32 emulation), TMEM chunk accumulators "
                 "flushed into round-to-nearest FP32 sums every 32 K-columns, TMA"
                 if engine == "tf32x3" else engine),
        "peak_source": (f"{peak_src}: bf16_tflops_sustained {bf16_sus:.0f} / 2 (TF32 rate) / 3 "
                        "(MMAs per FP32 product); sustained figure since the kernel runs inside "
                        "a long step"),
        "launches_per_step": d["launches"],
        "avg_launch_ms": d["ms"] / max(1, d["launches"]),
        "avg_sm_share": sm_share,
        "achieved_per_sm_share": achieved,
        "frac_per_sm_share": achieved / p32,
        "frac_note": ("frac = achieved / peak with achieved = flops / device span of the launches "
                      "(raw); *_per_sm_share divides by span x the SM share the co-scheduled "
                      "launch was given (its rate per whole-GPU equivalent)"),
        "algorithmic_flops_per_launch": d["flops"] / max(1, d["launches"]),
        "algorithmic_bytes_per_launch": d["bytes"] / max(1, d["launches"]),
        "measured": ("device-side %globaltimer span of every bulk trailing-update launch inside "
                     "the timed region (it runs concurrently with the co-scheduled FP64 band "
                     "update on the same stream, so stream events cannot bracket it); "
                     "algorithmic flops = reference flop model (factor.py:83-95) per launch"),
        "share_of_step": d["ms"] / (t_dev / args.steps * 1e3),
        "traffic_source": (f"profiles/ncu_traffic.json: ncu dram__bytes_read+write per bulk-update "
                           f"launch ({dom_kernel}, one evaluation at the bench config); above "
                           "the algorithmic C read+write because the A-panel row tiles are re-fetched "
                           "once per super-column of 12 output columns (DESIGN.md section 4)"),
        "cholesky_flop_weighted": {
            "roofline_ms": t_roof * 1e3, "achieved_ms": t_chol * 1e3, "frac": t_roof / t_chol,
            "f_sp": fl_plan.sp, "f_dp": fl_plan.dp,
            "p32_tflops": p32, "p64_tflops": p64,
            "p32_source": "MEASURED_PEAKS.json bf16_sustained/6 (3xTF32 on tcgen05)",
            "p64_burst_tflops": p64_burst, "p64_sustained_tflops": p64_sus,
            "p64_source": ("mt_peak_probe (csrc/prof.cu): independent FP64 DMMA m8n8k4 chains on "
                           "every SM, this run; burst = best single ~10 ms launch, sustained = "
                           "median launch over 4 s back to back (MEASURED_PEAKS.json has no "
                           "FP64 figure)")},
    }

    # ---- e2e through the public API from host buffers (pools of the timed
    #      evaluator freed first: MP at N=262144 needs ~145 GB)
    del ev
    _free_memory()
    e2e = None
    if not args.no_e2e:
        pin_locs = torch.from_numpy(np.array(ds.locations)).pin_memory()
        pin_z = torch.from_numpy(np.array(ds.z)).pin_memory()
        host_ds = mt.GeoDataset(pin_locs.numpy(), pin_z.numpy())

        def api_call():
            if dist_on:
                return loglik_distributed(host_ds, theta, nb, mp_pol, grid=grid)
            return mt.loglik(host_ds, theta, nb, mp_pol)

        k_e2e = max(1, min(args.steps, 2))
        barrier()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(st)
        for _ in range(k_e2e):
            out = api_call()
        s1.record(st)
        torch.cuda.synchronize()
        t_e2e = max_over_ranks(s0.elapsed_time(s1) / 1e3)
        e2e = {"value": k_e2e / t_e2e, "unit": UNIT,
               "h2d_bytes_per_step": int(ds.locations.nbytes + ds.z.nbytes),
               "d2h_bytes_per_step": 16 + 32 + 32,
               "api": ("paper_2003_05324_b200.distributed.loglik_distributed"
                       if dist_on else "paper_2003_05324_b200.loglik") +
                      "(dataset, params, nb, policy)",
               "loglik": out.value}
        _free_memory()

    # ---- the build's own full-DP path
    dp = None
    if not args.no_dp:
        p_tiles = -(-n // nb)
        dp_bytes = p_tiles * (p_tiles + 1) // 2 * nb * nb * 8 / world
        free_bytes = torch.cuda.mem_get_info()[0]
        free_min = -max_over_ranks(-float(free_bytes)) if dist_on else free_bytes
        # full DP at the headline N only when it fits and stays short (DMMA ~28 TF/s per
        # GPU under the power cap): 8 GPUs at N=262144 ~25 s; otherwise configs[1]
        dp_secs = (n ** 3 / 3.0) / (world * 28e12)
        if dp_bytes < 0.9 * free_min and dp_secs < 150.0:
            dn, dt, dasm, mp_ref = n, t, asm, value
        else:
            dn, dt = args.dp_n, args.dp_t
            dasm = mt.TileAssembler(_dataset(mt, dn), nb)
            evm = make_eval(dasm, mt.PrecisionPolicy.mp(diag_thick=dt))
            run_eval(evm, theta)
            barrier()
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(st)
            for _ in range(3):
                run_eval(evm, theta)
            a1.record(st)
            torch.cuda.synchronize()
            mp_ref = 3 / max_over_ranks(a0.elapsed_time(a1) / 1e3)
            del evm
            _free_memory()
        evd = make_eval(dasm, mt.PrecisionPolicy.dp())
        if dn != n:
            run_eval(evd, theta)  # warm (cheap at the reduced size)
        barrier()
        torch.cuda.synchronize()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(st)
        run_eval(evd, theta)
        d1.record(st)
        torch.cuda.synchronize()
        t_dp = max_over_ranks(d0.elapsed_time(d1) / 1e3)
        dp = {"n": dn, "mp_band_t": dt, "dp_evals_per_s": 1.0 / t_dp, "dp_ms_per_eval": t_dp * 1e3,
              "mp_evals_per_s": mp_ref, "mp_speedup": mp_ref * t_dp,
              "note": ("same N as the headline" if dn == n else
                       f"full DP at N={n} needs {dp_bytes * world / 1e9:.0f} GB and ~{dp_secs:.0f} s "
                       f"on {world} GPU(s): compared at configs[1] N={dn}")}
        del evd
        _free_memory()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_obj(args)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": warm,
            "ms_per_step": t_dev / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic",
            "config": {"workload": f"BASELINE metric config: N={n}, tile {nb}, MP band t={t}, "
                                   f"Matern{THETA}, one loglik evaluation per step",
                       "n": n, "nb": nb, "band_t": t, "theta": list(THETA),
                       "sp_flop_fraction": fl_plan.sp_fraction,
                       "l2": "inputs (tile pools, >= 35 GB) >> 126 MB L2; no flush needed",
                       "z": "N(0,1) timing-only observations (parity runs use field z)",
                       "parallelism": (f"2D block-cyclic {grid[0]}x{grid[1]} process grid, NCCL "
                                       f"row/column panel broadcasts" if dist_on else "1 GPU")},
            "cholesky_tflops": chol_tflops, "cholesky_ms": t_chol * 1e3,
            # per-kind event spans inside the timed region; panel-stream spans
            # include waiting for SMs held by the bulk update
            "kernel_event_spans_ms_per_step": {k: round(v["ms"], 3) for k, v in kinds.items()},
            "mp_vs_dp": dp, "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu,
            "gpu_launches": int(launches), "clocks": clocks.summary(),
            "library_options": opts or "defaults", "fp32_engine": engine,
            "nccl": ({"version": ".".join(map(str, torch.cuda.nccl.version())),
                      "world_size": world, "backend": dist.get_backend(),
                      "grid": list(grid),
                      "debug": (f"NCCL_DEBUG={os.environ.get('NCCL_DEBUG')} "
                                f"(INIT lines on stderr)")} if dist_on else None),
            "loglik_sample": results[-1],
        }
        print(json.dumps(line), flush=True)


def _free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(args):
    """`bench.py --gpus N` outside torchrun: re-launch this script as N ranks
    (one process per GPU) with torch.distributed.run on 127.0.0.1 and return
    its exit code.  Rank 0 prints the JSON line."""
    # the script's own flags travel in the environment: torchrun's parser would
    # claim abbreviations such as --n (--nnodes) or --t (--tee)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)]
    return subprocess.call(cmd, env=dict(os.environ, MT_BENCH_ARGV=json.dumps(sys.argv[1:])))


def nccl_debug_env():
    """NCCL's communicator-init lines (rank count, transports, NVLS) go to
    stderr, where the driver can count the ranks; stdout carries only the
    JSON line."""
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")


def run_dry(args, rank, world):
    """Launch/rendezvous check without a GPU (MT_BENCH_DRYRUN=1, gloo): every
    rank joins, the max-over-ranks reduction runs, rank 0 prints the line
    shape with n_gpus = world size.  Never used for reported numbers."""
    import torch
    import torch.distributed as dist
    seen = torch.tensor([1.0])
    t = torch.tensor([float(rank + 1)])
    if world > 1:
        dist.all_reduce(seen)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world,
                          "dry_run": True, "ranks_joined": int(seen.item()),
                          "max_over_ranks": t.item(), "steps": args.steps,
                          "warmup": args.warmup}), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if args.impl == "reference":  # the CPU arm is rank 0's alone; no ranks to spawn
            run_reference(args, 0)
            return
        sys.exit(spawn_ranks(args))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    dry = os.environ.get("MT_BENCH_DRYRUN") == "1"
    if world > 1:
        import torch
        import torch.distributed as dist
        if dry or os.environ.get("MT_BENCH_BACKEND", "nccl") == "gloo":
            # dev checks of the multi-rank logic: CPU-only (dry run) or ranks
            # sharing one GPU (NCCL refuses that); never used for reported numbers
            if not dry:
                torch.cuda.set_device(local_rank % torch.cuda.device_count())
            dist.init_process_group("gloo")
        else:
            nccl_debug_env()
            torch.cuda.set_device(local_rank % torch.cuda.device_count())
            # high-priority NCCL streams: the panel broadcasts get SMs ahead of the
            # bulk update's pending CTAs (which also yield on request)
            opts = dist.ProcessGroupNCCL.Options()
            opts.is_high_priority_stream = True
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank),
                                    pg_options=opts)
    if dry:
        run_dry(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
