"""Where the FP32 tcgen05 update's MMA issuer waits (dev tool, option 16)."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_05324_b200 as mt
from paper_2003_05324_b200 import _lib
lib = _lib.load()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
locs = mt.generate_locations(n, seed=mt.derive_seed(0, 0))
ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.random.default_rng(1).standard_normal(n)))
ev = mt.Evaluator(mt.TileAssembler(ds, 512), mt.PrecisionPolicy.mp(diag_thick=8))
th = mt.MaternParams(1.0, 0.1, 0.5)
ev(th)
for cfg in ({}, {17: 1}):
    olds = {k: lib.mt_set_option(k, v) for k, v in cfg.items()}
    lib.mt_set_option(16, 1)
    out = (ctypes.c_double * 4)()
    lib.mt_tcf_stats(out)
    e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    ev.launch(th, chol_events=e)
    ev.finish()
    lib.mt_tcf_stats(out)
    lib.mt_set_option(16, 0)
    for k, v in olds.items():
        lib.mt_set_option(k, v)
    tot = out[2]
    print(json.dumps({"n": n, "options": cfg, "cholesky_ms": e[0].elapsed_time(e[1]),
                      "issuers": out[3], "wait_operands_frac": out[0] / tot,
                      "wait_tmem_frac": out[1] / tot}), flush=True)
