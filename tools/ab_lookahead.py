"""Cholesky time with lookahead 1 vs 2 (dev tool)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_05324_b200 as mt
n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
locs = mt.generate_locations(n, seed=mt.derive_seed(0, 0))
ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.random.default_rng(1).standard_normal(n)))
asm = mt.TileAssembler(ds, 512)
th = mt.MaternParams(1.0, 0.1, 0.5)
for rnd in range(2):
    for la in (1, 2):
        ev = mt.Evaluator(asm, mt.PrecisionPolicy.mp(diag_thick=8), lookahead=la)
        ev(th)
        e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev.launch(th, chol_events=e)
        r = ev.finish()
        print(json.dumps({"n": n, "lookahead": la, "round": rnd, "cholesky_ms": e[0].elapsed_time(e[1]),
                          "logdet": r[0], "quad": r[1]}), flush=True)
        del ev
        torch.cuda.empty_cache()
