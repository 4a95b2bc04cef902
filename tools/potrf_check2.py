"""Cluster vs single-CTA POTRF inside full factorizations (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_05324_b200 as mt
from paper_2003_05324_b200 import _lib

lib = _lib.load()
for n, nb, pol in ((4096, 512, "mp:2"), (3000, 256, "dp"), (2048, 64, "mp:3"), (8192, 512, "mp:8")):
    locs = mt.generate_locations(n, seed=41)
    ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.zeros(n)))
    mode, _, t = pol.partition(":")
    policy = mt.PrecisionPolicy.dp() if mode == "dp" else mt.PrecisionPolicy.mp(diag_thick=int(t))
    res = []
    for flag in (0, 1, 1, 0):
        old = lib.mt_set_option(14, flag)
        try:
            f = mt.cholesky(mt.assemble_covariance(ds, mt.MaternParams(1.0, 0.1, 0.5), nb, policy))
            res.append(np.tril(f.matrix.to_dense()))
            print(n, nb, pol, flag, "ok", flush=True)
        except Exception as e:
            res.append(None)
            print(n, nb, pol, flag, "error", e, flush=True)
        finally:
            lib.mt_set_option(14, old)
    if all(r is not None for r in res):
        print("  diffs", [float(np.abs(r - res[0]).max()) for r in res[1:]], flush=True)
n, nb = 1024, 256
rng = np.random.default_rng(3)
x = rng.standard_normal((n, n))
a = x @ x.T / n + np.eye(n)
a[600, 600] = -5.0
for flag in (0, 1):
    old = lib.mt_set_option(14, flag)
    try:
        mt.cholesky(mt.TileMatrix.from_dense(a, nb, mt.PrecisionPolicy.dp()))
        print("npd: no error", flag)
    except mt.FactorizationError as e:
        print("npd index", flag, e.index)
    finally:
        lib.mt_set_option(14, old)
