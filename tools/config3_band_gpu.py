"""configs[2] band search on one B200 (dev tool): strong-correlation field
(beta=0.3, nu=1.0, Bessel path), N=131,072, nb=512.  z = the build's own
full-DP generate_field, then MP at the paper's DP-band tiers
(10/20/40/60/80% of p = 256: t = 26/51/102/154/205) with the default FP32
engine: NPD pivot or (Cholesky TF/s, speed-up vs own DP, loglik error vs DP).
One JSON line per band.

usage: python tools/config3_band_gpu.py [n] [engine]"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2003_05324_b200 as mt

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
eng = sys.argv[2] if len(sys.argv) > 2 else "tf32x3"
mt.set_fp32_engine(eng)
nb = 512
p = n // nb
th = mt.MaternParams(1.0, 0.3, 1.0)
locs = mt.generate_locations(n, seed=mt.derive_seed(3, 0))
ds, _ = mt.morton_sort(mt.generate_field(locs, th, seed=mt.derive_seed(3, 1), nb=nb))
asm = mt.TileAssembler(ds, nb)


def timed(pol):
    ev = mt.Evaluator(asm, pol)
    try:
        ev(th)
    except mt.FactorizationError as exc:
        del ev
        torch.cuda.empty_cache()
        return {"spd": False, "npd_index": exc.index}
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ev.launch(th, chol_events=(c0, c1))
    e1.record()
    ld, q = ev.finish()
    del ev
    torch.cuda.empty_cache()
    t_eval, t_chol = e0.elapsed_time(e1) / 1e3, c0.elapsed_time(c1) / 1e3
    return {"spd": True, "s_per_eval": t_eval, "cholesky_s": t_chol,
            "cholesky_tflops": n ** 3 / 3 / t_chol / 1e12,
            "loglik": -0.5 * (n * math.log(2 * math.pi) + ld + q), "quad_over_n": q / n}


dp = timed(mt.PrecisionPolicy.dp())
print(json.dumps({"n": n, "engine": eng, "policy": "dp", **dp}), flush=True)
for pct in (10, 20, 40, 60, 80):
    t = max(1, int(math.floor(p * pct / 100.0 + 0.5)))
    r = timed(mt.PrecisionPolicy.mp(diag_thick=t))
    if r["spd"]:
        r["speedup_vs_dp_eval"] = dp["s_per_eval"] / r["s_per_eval"]
        r["loglik_rel_err_vs_dp"] = abs(r["loglik"] - dp["loglik"]) / abs(dp["loglik"])
        fl = mt.planned_flops(n, nb, mt.PrecisionPolicy.mp(diag_thick=t))
        r["sp_flop_fraction"] = fl.sp_fraction
    print(json.dumps({"n": n, "engine": eng, "policy": f"mp:{pct}%", "t": t, **r}), flush=True)
