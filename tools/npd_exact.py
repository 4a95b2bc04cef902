"""Where does the MP factorization of the strong-correlation field break down
when the FP32 off-band GEMMs/TRSMs are correctly rounded (dev tool)?

The reference's MP algorithm (factor.py:230-285) stores every off-band result
in FP32.  Its NPD pivot also depends on how the FP32 products are summed
(OpenBLAS sgemm: sequential round-to-nearest FMA over K).  This runs the
oracle with the FP32 kernels replaced by correctly rounded ones -- operands
widened, product and update in FP64, ONE rounding to FP32 per output -- to
show which pivot the MP algorithm reaches when the summation adds no error.

usage: python tools/npd_exact.py [n] [t]     (defaults: 16384 8; nb 512)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from scipy.linalg import solve_triangular

from oracle import mixtile_oracle as O
import paper_2003_05324_b200.geodata as G


class _Exact:
    """scipy.linalg.blas stand-in: FP32 kernels correctly rounded, FP64 unchanged."""

    def __init__(self, blas):
        self._b = blas

    def __getattr__(self, name):
        return getattr(self._b, name)

    def sgemm(self, alpha, a, b, beta=1.0, c=None, trans_b=0, overwrite_c=0):
        a = np.asarray(a, np.float64)
        b = np.asarray(b, np.float64)
        prod = a @ (b.T if trans_b else b)
        return np.asfortranarray((beta * np.asarray(c, np.float64) + alpha * prod).astype(np.float32))

    def strsm(self, alpha, a, b, side=1, lower=1, trans_a=1, diag=0, overwrite_b=0):
        # B <- alpha B L^-T (side right, lower, transposed): X L^T = B
        a = np.asarray(a, np.float64)
        b = np.asarray(b, np.float64)
        x = solve_triangular(a, (alpha * b).T, lower=True).T
        return np.asfortranarray(x.astype(np.float32))


def npd_index(locs, theta, nb, t, blas=None):
    n = len(locs)
    p = -(-n // nb)
    saved = O._blas
    if blas is not None:
        O._blas = blas
    try:
        O.cholesky(O.assemble(locs, theta, nb, "mp", t), n, nb, "mp", t)
        return None
    except O.NotSPD as e:
        return e.index
    finally:
        O._blas = saved


if __name__ == "__main__":
    a = sys.argv[1:]
    n = int(a[0]) if a else 16384
    t = int(a[1]) if len(a) > 1 else 8
    nb, theta = 512, (1.0, 0.3, 1.0)
    locs = G.generate_locations(n, seed=G.derive_seed(3, 0))
    ds, _ = G.morton_sort(G.GeoDataset(locs, np.random.default_rng(3).standard_normal(n)))
    out = {"n": n, "nb": nb, "t": t, "theta": list(theta),
           "npd_reference_sgemm": npd_index(ds.locations, theta, nb, t),
           "npd_correctly_rounded_fp32": npd_index(ds.locations, theta, nb, t, _Exact(O._blas))}
    print(json.dumps(out), flush=True)
