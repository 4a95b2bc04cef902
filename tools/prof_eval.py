"""Run `warm` + `reps` likelihood evaluations of one config (ncu capture target)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_05324_b200 as mt

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--nb", type=int, default=512)
ap.add_argument("--t", type=int, default=2)
ap.add_argument("--dp", action="store_true")
ap.add_argument("--warm", type=int, default=1)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
if os.environ.get("MT_OPTS"):  # e.g. MT_OPTS=10=0 (library runtime options)
    from paper_2003_05324_b200 import _lib
    for kv in os.environ["MT_OPTS"].split(","):
        k_, v_ = kv.split("=")
        _lib.load().mt_set_option(int(k_), int(v_))
locs = mt.generate_locations(a.n, seed=mt.derive_seed(0, 0))
ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.random.default_rng(1).standard_normal(a.n)))
pol = mt.PrecisionPolicy.dp() if a.dp else mt.PrecisionPolicy.mp(diag_thick=a.t)
ev = mt.Evaluator(mt.TileAssembler(ds, a.nb), pol)
th = mt.MaternParams(1.0, 0.1, 0.5)
for _ in range(a.warm + a.reps):
    print(ev(th), flush=True)
