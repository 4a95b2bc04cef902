"""Profile log-likelihood along a line through the DP optimum of the configs[4]
dataset (N=65,536): full DP vs MP t=2 with the tcgen05 3xTF32 engine and with
the SIMT FFMA (round-to-nearest) engine.  Shows how smooth MP(theta) - DP(theta)
is -- what the Nelder-Mead driver sees (dev tool)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_05324_b200 as mt

n, nb = 65536, 512
theta = mt.MaternParams(1.0, 0.1, 0.5)
locs = mt.generate_locations(n, seed=mt.derive_seed(5, 0))
ds, _ = mt.morton_sort(mt.generate_field(locs, theta, seed=mt.derive_seed(5, 1), nb=nb))
asm = mt.TileAssembler(ds, nb)
nu = 0.49685
betas = np.linspace(0.0870, 0.0886, 9)
rows = {}
T = int(os.environ.get("T", 2))
for tag, pol, eng in (("dp", mt.PrecisionPolicy.dp(), "tf32x3"),
                      ("mp_tf32x3", mt.PrecisionPolicy.mp(diag_thick=T), "tf32x3"),
                      ("mp_ffma", mt.PrecisionPolicy.mp(diag_thick=T), "ffma")):
    mt.set_fp32_engine(eng)
    ev = mt.Evaluator(asm, pol)
    vals = []
    for b in betas:
        ld, q = ev(mt.MaternParams(1.0, float(b), nu))
        vals.append(mt.mle._profile_from(n, ld, q).value)
    rows[tag] = vals
mt.set_fp32_engine("tf32x3")
dp = np.array(rows["dp"])
out = {"band_t": T, "betas": betas.tolist(), "nu": nu, "dp": rows["dp"]}
for tag in ("mp_tf32x3", "mp_ffma"):
    d = np.array(rows[tag]) - dp
    out[tag + "_minus_dp"] = d.tolist()
    # roughness: residual of a quadratic fit of the difference in beta
    c = np.polyfit(betas, d, 2)
    out[tag + "_rough"] = float(np.std(d - np.polyval(c, betas)))
    out[tag + "_argmax_beta"] = float(betas[int(np.argmax(rows[tag]))])
out["dp_argmax_beta"] = float(betas[int(np.argmax(dp))])
print(json.dumps(out))
