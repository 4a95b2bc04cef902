"""Which MP component moves kriging away from DP (dev tool): FP32 engine x TRSM variant."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_05324_b200 as mt
from oracle import mixtile_oracle as O

for n, nb, t in ((2048, 256, 2), (4096, 512, 2), (4096, 256, 4)):
    th = (1.0, 0.1, 0.5)
    ds = mt.generate_field(mt.generate_locations(n, seed=21), mt.MaternParams(*th), seed=22)
    test = mt.generate_locations(300, seed=23)
    want_dp = O.krige(ds.locations, ds.z, test, th, nb, "dp", n // nb)
    want_mp = O.krige(ds.locations, ds.z, test, th, nb, "mp", t)
    out = [f"n={n} nb={nb} t={t}: cpuMP gap {np.max(np.abs(want_mp - want_dp)):.2e}"]
    for eng, tct in (("ffma", 0), ("tf32x3", 0), ("tf32x3", 1)):
        mt.set_fp32_engine(eng); mt.set_tc_trsm(tct)
        got = mt.krige(ds, test, mt.MaternParams(*th), nb, mt.PrecisionPolicy.mp(diag_thick=t))
        out.append(f"{eng}/tctrsm={tct} {np.max(np.abs(got - want_dp)):.2e}")
    mt.set_fp32_engine("tf32x3"); mt.set_tc_trsm(1)
    print("  ".join(out), flush=True)
