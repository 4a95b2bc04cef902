"""FP32 engine accuracy + speed on the GPU (dev tool): 'ffma' (SIMT, RN),
'tf32x3' (tcgen05 3xTF32, RN chunk accumulation, default) and 'tf32x3_rz'
(whole-K TMEM accumulation, RZ).  Prints one JSON line per engine.

usage: python tools/acc_engines.py [--no-time] [--n-time 65536]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2003_05324_b200 as mt
from oracle import mixtile_oracle as O

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import load_golden  # noqa: E402

ENGINES = ("ffma", "tf32x3", "tf32x3_rz")
args = sys.argv[1:]
n_time = int(args[args.index("--n-time") + 1]) if "--n-time" in args else 65536

# 1. factor error vs the oracle's MP factor (tests/test_gpu_tc.py setup)
n, nb, t, th = 2048, 256, 2, (1.0, 0.1, 0.5)
ds1, _ = mt.morton_sort(mt.GeoDataset(mt.generate_locations(n, seed=3), np.zeros(n)))
ref = O.cholesky(O.assemble(ds1.locations, th, nb, "mp", t), n, nb, "mp", t)
# 2. kriging (tests/test_gpu_predict.py::test_krige_vs_oracle_larger setup)
dsk = mt.generate_field(mt.generate_locations(2048, seed=21), mt.MaternParams(*th), seed=22)
test = mt.generate_locations(300, seed=23)
kdp = O.krige(dsk.locations, dsk.z, test, th, 256, "dp", 8)
kmp = O.krige(dsk.locations, dsk.z, test, th, 256, "mp", 2)
kgap = float(np.max(np.abs(kmp - kdp)))
# 3. strong-correlation golden (reference-generated)
gs = load_golden("strong1024")
dss = mt.GeoDataset(gs["locs"], gs["z"])
ths = mt.MaternParams(*gs["theta"])
# 4. strong16384 NPD index
g16 = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                  "tests", "golden", "strong16384_npd.json")))
loc16 = mt.generate_locations(g16["n"], seed=mt.derive_seed(3, 0))
ds16, _ = mt.morton_sort(mt.GeoDataset(loc16, np.random.default_rng(3).standard_normal(g16["n"])))

out = {}
for eng in (() if "--only-time" in args else ENGINES):
    mt.set_fp32_engine(eng)
    r = {"engine": eng}
    f = mt.cholesky(mt.assemble_covariance(ds1, mt.MaternParams(*th), nb, mt.PrecisionPolicy.mp(diag_thick=t)))
    r["factor_err_vs_oracle_mp"] = max(float(np.max(np.abs(f.tiles[k].dp - v[0]))) for k, v in ref.items())
    kp = mt.krige(dsk, test, mt.MaternParams(*th), 256, mt.PrecisionPolicy.mp(diag_thick=2))
    r["krige_dev_from_dp"] = float(np.max(np.abs(kp - kdp)))
    r["krige_dev_over_reference_gap"] = r["krige_dev_from_dp"] / kgap
    dp_val = gs["results"]["dp"][0]
    st = {}
    for tag, want in gs["results"].items():
        if tag == "dp" or want[0] == "npd":
            continue
        ev = mt.loglik(dss, ths, int(gs["nb"]), mt.PrecisionPolicy.mp(diag_thick=int(tag.split(":")[1])))
        st[tag] = {"rel_vs_cpu_mp": abs(ev.value - want[0]) / abs(want[0]),
                   "gpu_rel_vs_dp": abs(ev.value - dp_val) / abs(dp_val),
                   "cpu_rel_vs_dp": abs(want[0] - dp_val) / abs(dp_val)}
    r["strong1024"] = st
    try:
        mt.loglik(ds16, mt.MaternParams(*g16["theta"]), g16["nb"], mt.PrecisionPolicy.mp(diag_thick=g16["band_t"]))
        r["strong16384_npd_index"] = None
    except mt.FactorizationError as e:
        r["strong16384_npd_index"] = e.index
    r["reference_npd_index"] = g16["reference_factorization_error_index"]
    out[eng] = r
    print(json.dumps(r), flush=True)

if "--no-time" not in args:
    dst = mt.generate_locations(n_time, seed=mt.derive_seed(0, 0))
    dst, _ = mt.morton_sort(mt.GeoDataset(dst, np.random.default_rng(1).standard_normal(n_time)))
    for t_band in (8, 2):
        for eng in ENGINES:
            mt.set_fp32_engine(eng)
            ev = mt.Evaluator(mt.TileAssembler(dst, 512), mt.PrecisionPolicy.mp(diag_thick=t_band))
            th0 = mt.MaternParams(1.0, 0.1, 0.5)
            ev(th0)
            torch.cuda.synchronize()
            best = 1e9
            for _ in range(3):
                e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                ev.launch(th0, chol_events=e)
                res = ev.finish()
                best = min(best, e[0].elapsed_time(e[1]))
            print(json.dumps({"engine": eng, "n": n_time, "t": t_band, "cholesky_ms": best,
                              "tflops": n_time ** 3 / 3 / best / 1e9,
                              "loglik": -0.5 * (n_time * np.log(2 * np.pi) + res[0] + res[1])}), flush=True)
            del ev
            torch.cuda.empty_cache()
    mt.set_fp32_engine("tf32x3")
