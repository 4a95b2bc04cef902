"""BASELINE configs[2] on one B200: strong-correlation field (beta=0.3, nu=1.0,
Bessel path) at N=131,072, nb=512, MP band t=8 vs the build's own full DP.
One JSON line: seconds per evaluation / Cholesky TF/s for both, MP speed-up,
loglik relative difference (timing-only z ~ N(0,1))."""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_05324_b200 as mt

n, nb, t = int(os.environ.get("N", 131072)), 512, 8
th = mt.MaternParams(1.0, 0.3, 1.0)
locs = mt.generate_locations(n, seed=mt.derive_seed(3, 0))
ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.random.default_rng(3).standard_normal(n)))
asm = mt.TileAssembler(ds, nb)
out = {"config": f"configs[2]: N={n}, nb={nb}, theta={th.as_tuple()} (Bessel K_nu path), 1 GPU"}
for tag, pol in (("mp_t8", mt.PrecisionPolicy.mp(diag_thick=t)), ("dp", mt.PrecisionPolicy.dp())):
    ev = mt.Evaluator(asm, pol)
    try:
        ev(th)  # warm
    except mt.FactorizationError as exc:
        out[tag] = {"not_positive_definite_at": exc.index}
        del ev
        torch.cuda.empty_cache()
        continue
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ev.launch(th, chol_events=(c0, c1))
    e1.record()
    ld, q = ev.finish()
    t_eval, t_chol = e0.elapsed_time(e1) / 1e3, c0.elapsed_time(c1) / 1e3
    out[tag] = {"s_per_eval": t_eval, "cholesky_s": t_chol, "cholesky_tflops": n ** 3 / 3 / t_chol / 1e12,
                "loglik": -0.5 * (n * math.log(2 * math.pi) + ld + q)}
    del ev
    torch.cuda.empty_cache()
if "s_per_eval" in out["dp"] and "s_per_eval" in out["mp_t8"]:
    out["mp_speedup_eval"] = out["dp"]["s_per_eval"] / out["mp_t8"]["s_per_eval"]
    out["mp_speedup_cholesky"] = out["dp"]["cholesky_s"] / out["mp_t8"]["cholesky_s"]
    out["loglik_rel_diff"] = abs(out["mp_t8"]["loglik"] - out["dp"]["loglik"]) / abs(out["dp"]["loglik"])
print(json.dumps(out))
