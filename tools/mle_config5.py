"""BASELINE configs[4] on one B200: Matern MLE at N=65,536 (nb=512), mixed
precision (bands BANDS, default 2) vs the build's own full DP, on one field-sampled dataset.
Prints one JSON object (theta-hat per precision, relative differences,
evaluations, seconds).  The CPU reference cannot run this size (SURVEY.md
8d); its agreement is tested at small N (tests/test_gpu_mle.py)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_05324_b200 as mt

n, nb = int(os.environ.get("N", 65536)), 512
theta = mt.MaternParams(1.0, 0.1, 0.5)
locs = mt.generate_locations(n, seed=mt.derive_seed(5, 0))
ds, _ = mt.morton_sort(mt.generate_field(locs, theta, seed=mt.derive_seed(5, 1), nb=nb))
out = {"config": f"configs[4]: MLE at N={n}, nb={nb}, field theta={theta.as_tuple()}, seed 5",
       "optimizer": "reference Nelder-Mead on log(range, smoothness), profiled variance (mle.py:131-224)"}
fits = {}
bands = [int(x) for x in os.environ.get("BANDS", "2").split(",")]
pols = [(f"mp_t{t}", mt.PrecisionPolicy.mp(diag_thick=t)) for t in bands] + [("dp", mt.PrecisionPolicy.dp())]
for tag, pol in pols:
    t0 = time.perf_counter()
    res = mt.fit_matern(ds, nb, pol)
    dt = time.perf_counter() - t0
    fits[tag] = res
    out[tag] = {"theta_hat": list(res.params.as_tuple()), "loglik": res.value,
                "evaluations": res.evaluations, "iterations": res.iterations,
                "converged": res.converged, "seconds": dt, "s_per_eval": dt / res.evaluations}
b = np.array(fits["dp"].params.as_tuple())
for t in bands:
    a = np.array(fits[f"mp_t{t}"].params.as_tuple())
    rel = np.abs(a - b) / np.abs(b)
    out[f"mp_t{t}_vs_dp_rel_diff"] = rel.tolist()
    # literally: each parameter rounds to the same 3 significant digits
    out[f"mp_t{t}_3sig"] = [[f"{x:.3g}", f"{y:.3g}"] for x, y in zip(a, b)]
    out[f"mp_t{t}_agree_3_significant_digits"] = all(f"{x:.3g}" == f"{y:.3g}" for x, y in zip(a, b))
    out[f"mp_t{t}_speedup_per_eval"] = out["dp"]["s_per_eval"] / out[f"mp_t{t}"]["s_per_eval"]
print(json.dumps(out))
if os.environ.get("SAVE"):  # inputs + GPU fits for the CPU reference loglik at theta-hat
    np.savez_compressed(os.environ["SAVE"], locs=ds.locations, z=ds.z, nb=np.array(nb),
                        fits=np.array(json.dumps(out)))
