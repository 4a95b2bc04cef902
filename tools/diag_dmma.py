"""Compare the TMA DMMA band update against the register-staged one (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_05324_b200 as mt

for n, nb, t in [(4096, 256, 8), (8192, 512, 4), (8192, 512, 8), (16384, 512, 8), (8192, 512, 2)]:
    locs = mt.generate_locations(n, seed=5)
    ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.zeros(n)))
    pol = mt.PrecisionPolicy.mp(diag_thick=t)
    out = []
    for legacy in (1, 0):
        mt.set_legacy_dmma(legacy)
        m = mt.assemble_covariance(ds, mt.MaternParams(1.0, 0.1, 0.5), nb, pol)
        # one step of updates only: potrf/trsm(0) + update(0) via lookahead-0 factor is the
        # whole thing; compare full factors
        try:
            f = mt.cholesky(m, lookahead=0)
            out.append({k: (v.dp.copy() if v.dp is not None else None) for k, v in f.tiles.items()})
        except Exception as e:
            out.append(str(e))
    mt.set_legacy_dmma(0)
    if isinstance(out[1], str) or isinstance(out[0], str):
        print(n, nb, t, "error", out[0] if isinstance(out[0], str) else "", out[1] if isinstance(out[1], str) else "")
        continue
    bad = []
    for key in sorted(out[0]):
        a, b = out[0][key], out[1][key]
        if a is None or b is None:
            continue
        if not np.array_equal(a, b):
            d = np.abs(a - b)
            r, c = np.unravel_index(np.argmax(d), d.shape)
            bad.append((key, float(d.max()), int(r), int(c)))
    print(n, nb, t, "mismatching tiles:", len(bad), bad[:8], flush=True)
