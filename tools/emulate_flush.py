"""CPU emulation (dev tool) of the 3xTF32 tcgen05 update with the TMEM
accumulator flushed every L k-steps into a round-to-nearest FP32 running sum
(registers), C <- RN(C - sum) at the end.  Compares kriging / loglik
deviation from DP against the reference sgemm (RN) and the unflushed RZ engine.

usage: python tools/emulate_flush.py [n] [nb] [t] [beta] [nu]"""
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


def make(flush, order="lhm"):
    """flush = k-steps (K=8 each) per TMEM chunk; 0 = never (today's engine)."""
    def sgemm(alpha, a, b, beta=1.0, c=None, trans_b=0, overwrite_c=0):
        a = np.asarray(a, np.float32); b = np.asarray(b, np.float32)
        ah = tf32(a, "rna"); al = tf32(a - ah, "trunc")
        bh = tf32(b, "rna"); bl = tf32(b - bh, "trunc")
        m, K = a.shape; n = b.shape[0]
        f = lambda x: x.astype(np.float64)
        acc = np.zeros((m, n), np.float32)
        tot = np.zeros((m, n), np.float32)
        steps = K // 8
        for s_i, k0 in enumerate(range(0, K, 8)):
            s = slice(k0, k0 + 8)
            for x, y in ((al, bh), (ah, bl), (ah, bh)):
                acc = rz32(f(acc) + f(x[:, s]) @ f(y[:, s]).T)
            if flush and ((s_i + 1) % flush == 0 or s_i == steps - 1):
                tot = (f(tot) + f(acc)).astype(np.float32)
                acc[:] = 0
        if not flush:
            tot = acc
        return np.asfortranarray((np.asarray(c, np.float64) - f(tot)).astype(np.float32))
    return sgemm


if __name__ == "__main__":
    a = sys.argv[1:]
    n = int(a[0]) if a else 2048
    nb = int(a[1]) if len(a) > 1 else 256
    t = int(a[2]) if len(a) > 2 else 2
    th = (1.0, float(a[3]) if len(a) > 3 else 0.1, float(a[4]) if len(a) > 4 else 0.5)
    locs = G.generate_locations(n, seed=21)
    if os.environ.get("SORT"): locs = locs[np.argsort(G.morton_keys(locs), kind="stable")]
    fac = O.cholesky(O.assemble(locs, th, nb, "dp", n // nb), n, nb, "dp", n // nb)
    z = O.matvec_lower(fac, n, nb, np.random.default_rng(22).standard_normal(n))
    test = G.generate_locations(300, seed=23)
    dp = O.krige(locs, z, test, th, nb, "dp", n // nb)
    ld_dp = O.loglik(locs, z, th, nb, "dp", n // nb)[0]
    cases = [("sgemm RN (reference)", _orig)] + [
        (f"3xTF32 RZ flush {L:>2d} k-steps" if L else "3xTF32 RZ unflushed", make(L))
        for L in (0, 32, 16, 8, 4, 2, 1)]
    for name, fn in cases:
        O._blas.sgemm = fn
        mp = O.krige(locs, z, test, th, nb, "mp", t)
        ld = O.loglik(locs, z, th, nb, "mp", t)[0]
        print(f"{name:30s} krige |mp-dp| {np.max(np.abs(mp - dp)):.2e}   loglik rel "
              f"{abs(ld - ld_dp) / abs(ld_dp):.2e}", flush=True)
    O._blas.sgemm = _orig
