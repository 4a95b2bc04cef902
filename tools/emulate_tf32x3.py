"""CPU emulation of the tcgen05 3xTF32 FP32 update inside the oracle's MP
Cholesky (dev tool): which rounding effect moves kriging away from DP?

sgemm in the oracle is replaced by C - sum_k8 MMA(..) with exact products,
the K=8 partial added to an FP32 accumulator with round-to-nearest (RN) or
round-toward-zero (RZ), lo operands truncated or rounded to TF32."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import mixtile_oracle as O
import paper_2003_05324_b200.geodata as G

_orig = O._blas.sgemm


def rz32(x):
    y = x.astype(np.float32)
    over = np.abs(y.astype(np.float64)) > np.abs(x)
    y[over] = np.nextafter(y[over], np.float32(0))
    return y


def tf32(x, mode):
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    if mode == "rna":
        u = (u + np.uint32(0x1000)) & np.uint32(0xFFFFE000)
    else:
        u = u & np.uint32(0xFFFFE000)
    return u.view(np.float32)


def make(acc_mode, lo_mode, split):
    def sgemm(alpha, a, b, beta=1.0, c=None, trans_b=0, overwrite_c=0):
        a = np.asarray(a, np.float32); b = np.asarray(b, np.float32)
        ah = tf32(a, "rna"); al = tf32(a - ah, lo_mode)
        bh = tf32(b, "rna"); bl = tf32(b - bh, lo_mode)
        m, K = a.shape; n = b.shape[0]
        rnd = rz32 if acc_mode == "rz" else (lambda x: x.astype(np.float32))
        acc = np.zeros((m, n), np.float32); corr = np.zeros((m, n), np.float32)
        f = lambda x: x.astype(np.float64)
        for k0 in range(0, K, 8):
            s = slice(k0, k0 + 8)
            for x, y, main in ((al, bh, False), (ah, bl, False), (ah, bh, True)):
                part = f(x[:, s]) @ f(y[:, s]).T
                if split and not main:
                    corr = rnd(f(corr) + part)
                else:
                    acc = rnd(f(acc) + part)
        tot = (acc.astype(np.float64) + corr) if split else acc.astype(np.float64)
        if split:
            tot = tot.astype(np.float32).astype(np.float64)
        return np.asfortranarray((np.asarray(c, np.float64) - tot).astype(np.float32))
    return sgemm


n, nb, t = int(sys.argv[1]) if len(sys.argv) > 1 else 2048, 256, 2
th = (1.0, 0.1, 0.5)
locs = G.generate_locations(n, seed=21)
# field z from the oracle's own DP factor
fac = O.cholesky(O.assemble(locs, th, nb, "dp", n // nb), n, nb, "dp", n // nb)
z = O.matvec_lower(fac, n, nb, np.random.default_rng(22).standard_normal(n))
test = G.generate_locations(300, seed=23)
dp = O.krige(locs, z, test, th, nb, "dp", n // nb)
ld_dp = O.loglik(locs, z, th, nb, "dp", n // nb)[0]
for name, fn in [("sgemm RN (reference)", _orig), ("3xTF32 acc RN, lo trunc", make("rn", "trunc", False)),
                 ("3xTF32 acc RZ, lo trunc", make("rz", "trunc", False)),
                 ("3xTF32 acc RZ, lo rna", make("rz", "rna", False)),
                 ("3xTF32 acc RZ, split main/corr", make("rz", "trunc", True))]:
    O._blas.sgemm = fn
    mp = O.krige(locs, z, test, th, nb, "mp", t)
    ld = O.loglik(locs, z, th, nb, "mp", t)[0]
    print(f"{name:34s} krige |mp-dp| {np.max(np.abs(mp - dp)):.2e}   loglik rel {abs(ld - ld_dp) / abs(ld_dp):.2e}", flush=True)
O._blas.sgemm = _orig
