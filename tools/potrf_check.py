"""Cluster vs single-CTA POTRF on single tiles (dev tool): max |diff| per 32x32 block."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_05324_b200 as mt
from paper_2003_05324_b200 import _lib

lib = _lib.load()
for n, nb in ((512, 512), (256, 256), (1024, 256), (96, 96), (128, 64)):
    rng = np.random.default_rng(n + nb)
    x = rng.standard_normal((n, n))
    a = x @ x.T / n + np.eye(n)
    outs = []
    for flag in (0, 1):
        old = lib.mt_set_option(14, flag)
        try:
            f = mt.cholesky(mt.TileMatrix.from_dense(a, nb, mt.PrecisionPolicy.dp()))
            outs.append(np.tril(f.matrix.to_dense()))
        except Exception as e:
            outs.append(None)
            print(n, nb, flag, "error", e)
        finally:
            lib.mt_set_option(14, old)
    if outs[0] is not None and outs[1] is not None:
        d = np.abs(outs[0] - outs[1])
        want = np.linalg.cholesky(a)
        bad = [(i, j) for i in range(0, n, 32) for j in range(0, i + 1, 32)
               if d[i:i + 32, j:j + 32].max() > 0]
        print(n, nb, "maxdiff", d.max(), "err_single", np.abs(outs[0] - want).max(),
              "err_cluster", np.abs(outs[1] - want).max(), "blocks differing", bad[:12])
