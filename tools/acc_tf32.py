"""Accuracy of the FP32 off-band engines vs the CPU oracle (dev tool):
max |L_gpu - L_oracle| over the factor for SIMT FFMA and tcgen05 3xTF32,
and the MP loglik relative error vs the oracle's MP and DP."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_05324_b200 as mt
from oracle import mixtile_oracle as O

print("lib:", os.environ.get("MIXTILE_LIB", "default"))
for n, nb, t, theta in ((2048, 256, 2, (1.0, 0.1, 0.5)), (4096, 512, 2, (1.0, 0.1, 0.5)),
                        (4096, 256, 1, (1.0, 0.3, 1.0))):
    locs = mt.generate_locations(n, seed=3)
    ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.random.default_rng(4).standard_normal(n)))
    ref = O.cholesky(O.assemble(ds.locations, theta, nb, "mp", t), n, nb, "mp", t)
    ref_dp = O.cholesky(O.assemble(ds.locations, theta, nb, "dp", n // nb), n, nb, "dp", n // nb)
    errs = {}
    for eng in ("ffma", "tf32x3"):
        mt.set_fp32_engine(eng)
        f = mt.cholesky(mt.assemble_covariance(ds, mt.MaternParams(*theta), nb,
                                               mt.PrecisionPolicy.mp(diag_thick=t)))
        e_mp = max(float(np.max(np.abs(f.tiles[key].dp - dp))) for key, (dp, _) in ref.items())
        e_dp = max(float(np.max(np.abs(f.tiles[key].dp - dp))) for key, (dp, _) in ref_dp.items())
        ev = mt.loglik(ds, mt.MaternParams(*theta), nb, mt.PrecisionPolicy.mp(diag_thick=t))
        errs[eng] = (e_mp, e_dp, ev.value)
    mt.set_fp32_engine("tf32x3")
    cpu_mp = O.loglik(ds.locations, ds.z, theta, nb, "mp", t)[0]
    cpu_dp = O.loglik(ds.locations, ds.z, theta, nb, "dp", n // nb)[0]
    e_cpu = max(float(np.max(np.abs(ref[key][0] - dp))) for key, (dp, _) in ref_dp.items())
    print(f"n={n} nb={nb} t={t} theta={theta}: |L-L_cpuMP| ffma {errs['ffma'][0]:.2e} tf32x3 "
          f"{errs['tf32x3'][0]:.2e} (ratio {errs['tf32x3'][0] / errs['ffma'][0]:.2f}); |L-L_DP| "
          f"cpuMP {e_cpu:.2e} ffma {errs['ffma'][1]:.2e} tf32x3 {errs['tf32x3'][1]:.2e}")
    print(f"   loglik rel vs cpuMP: ffma {abs(errs['ffma'][2] - cpu_mp) / abs(cpu_mp):.2e} tf32x3 "
          f"{abs(errs['tf32x3'][2] - cpu_mp) / abs(cpu_mp):.2e}; vs DP: cpuMP "
          f"{abs(cpu_mp - cpu_dp) / abs(cpu_dp):.2e} ffma {abs(errs['ffma'][2] - cpu_dp) / abs(cpu_dp):.2e} "
          f"tf32x3 {abs(errs['tf32x3'][2] - cpu_dp) / abs(cpu_dp):.2e}", flush=True)
