"""configs[2] (strong correlation, beta=0.3, nu=1.0): which DP band keeps the
MP factorization positive definite?  CPU half, on the oracle port of the
reference (dev tool): for each N, assemble the covariance once in FP64
(Bessel path, covmath.py:186-212), factor it in DP, draw z = L v, then run the
reference's MP algorithm at the paper's 10/20/40% DP-band tiers
(t = percent_to_thickness(pct, p), tilestore.py:33-43) and
record the NPD pivot or the loglik error against DP.

usage: python tools/config3_bands.py <n> [<n> ...]   (nb 512)"""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import mixtile_oracle as O
import paper_2003_05324_b200.geodata as G

THETA = (1.0, 0.3, 1.0)
NB = 512


def run(n):
    p = -(-n // NB)
    locs = G.generate_locations(n, seed=G.derive_seed(3, 0))
    ds, _ = G.morton_sort(G.GeoDataset(locs, np.zeros(n)))
    t0 = time.perf_counter()
    full = O.assemble(ds.locations, THETA, NB, "dp", p)
    t_asm = time.perf_counter() - t0
    fac = O.cholesky(full, n, NB, "dp", p)
    z = O.matvec_lower(fac, n, NB, np.random.default_rng(G.derive_seed(3, 1)).standard_normal(n))
    ld = O.logdet(fac, p)
    q = float(z @ O.solve(fac, n, NB, z))
    l_dp = -0.5 * (n * O.LOG_2PI + ld + q)
    del fac
    out = {"n": n, "nb": NB, "p": p, "theta": list(THETA), "assemble_s": t_asm, "dp_loglik": l_dp,
           "z_seed": "z = L_dp v, v = default_rng(derive_seed(3, 1)).standard_normal(n)", "mp": {}}
    for pct in (10, 20, 40):
        t = O.thickness("mp", p, dp_percent=pct)
        tiles = {k: (a if k[0] - k[1] < t else O.narrow(a)) for k, a in full.items()}
        t1 = time.perf_counter()
        try:
            f = O.cholesky(tiles, n, NB, "mp", t)
            ldm = O.logdet(f, p)
            qm = float(z @ O.solve(f, n, NB, z))
            lm = -0.5 * (n * O.LOG_2PI + ldm + qm)
            rec = {"t": t, "spd": True, "loglik": lm, "rel_err_vs_dp": abs(lm - l_dp) / abs(l_dp)}
            del f
        except O.NotSPD as e:
            rec = {"t": t, "spd": False, "npd_index": e.index}
        rec["seconds"] = time.perf_counter() - t1
        out["mp"][f"{pct}%"] = rec
        print(json.dumps({"n": n, "pct": pct, **rec}), flush=True)
    return out


if __name__ == "__main__":
    res = [run(int(a)) for a in (sys.argv[1:] or ["16384"])]
    print(json.dumps(res), flush=True)
