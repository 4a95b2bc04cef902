"""BASELINE configs[1] on one B200: N=65,536, nb=512, DP-band width sweep
(t = 1, 2, 4, 8, full DP) on a field-sampled z (the build's own full-DP
generate_field): Cholesky seconds / TF/s and loglik relative error vs full DP."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_05324_b200 as mt

n, nb = 65536, 512
th = mt.MaternParams(1.0, 0.1, 0.5)
locs = mt.generate_locations(n, seed=mt.derive_seed(0, 0))
ds, _ = mt.morton_sort(mt.generate_field(locs, th, seed=mt.derive_seed(0, 1), nb=nb))
asm = mt.TileAssembler(ds, nb)
rows = {}
for t in (1, 2, 4, 8, asm.p):
    pol = mt.PrecisionPolicy.dp() if t == asm.p else mt.PrecisionPolicy.mp(diag_thick=t)
    ev = mt.Evaluator(asm, pol)
    ev(th)
    best = None
    for _ in range(2):
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); ev.launch(th, chol_events=(c0, c1)); e1.record()
        ld, q = ev.finish()
        tc, te = c0.elapsed_time(c1) / 1e3, e0.elapsed_time(e1) / 1e3
        best = (tc, te) if best is None or tc < best[0] else best
    fl = mt.planned_flops(n, nb, pol)
    rows["dp" if t == asm.p else f"mp_t{t}"] = {
        "cholesky_s": best[0], "eval_s": best[1], "cholesky_tflops": n ** 3 / 3 / best[0] / 1e12,
        "sp_flop_fraction": fl.sp_fraction, "loglik": -0.5 * (n * math.log(2 * math.pi) + ld + q)}
    del ev
    torch.cuda.empty_cache()
dp = rows["dp"]
for k, v in rows.items():
    v["loglik_rel_err_vs_dp"] = abs(v["loglik"] - dp["loglik"]) / abs(dp["loglik"])
    v["speedup_vs_dp"] = dp["eval_s"] / v["eval_s"]
print(json.dumps({"config": "configs[1]: N=65536, nb=512, theta=(1, 0.1, 0.5), field-sampled z", **rows}))
