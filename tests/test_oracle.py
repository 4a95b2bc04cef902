"""CPU: the oracle restatement is pinned to the reference's own outputs.

tests/golden/*.npz were produced by running the real reference
(tests/golden/make_golden.py).  The oracle uses the same LAPACK/BLAS calls,
so likelihoods must agree BITWISE; special functions to the reference's own
test tolerances (test_covmath.py).
"""

import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, tag_to_mode
from oracle import mixtile_oracle as O


@pytest.mark.parametrize("name", ["config1", "strong1024", "ragged1000"])
def test_oracle_loglik_bitwise_vs_reference(name):
    g = load_golden(name)
    nb = int(g["nb"])
    n = len(g["z"])
    p = -(-n // nb)
    for tag, want in g["results"].items():
        mode, t = tag_to_mode(tag, p)
        if want[0] == "npd":
            with pytest.raises(O.NotSPD) as exc:
                O.loglik(g["locs"], g["z"], tuple(g["theta"]), nb, mode, t)
            assert exc.value.index == want[1]
            continue
        val, ld, q = O.loglik(g["locs"], g["z"], tuple(g["theta"]), nb, mode, t)
        assert (val, ld, q) == tuple(want), (name, tag)


def test_oracle_known_answers():
    # test_mle.py:36-50 (n = 1, z = 0) and two decorrelated points
    v, ld, q = O.loglik(np.array([[0.5, 0.5]]), np.array([0.0]), (1.0, 0.1, 0.5), 16, "dp", 1)
    assert math.isclose(v, -0.9189385332046727, rel_tol=0, abs_tol=1e-15)
    v, ld, q = O.loglik(np.array([[0.1, 0.1], [0.9, 0.9]]), np.array([1.0, 1.0]),
                        (1.0, 1e-3, 0.5), 16, "dp", 1)
    assert math.isclose(v, -2.8378770664093453, rel_tol=0, abs_tol=1e-14) and q == 2.0
    pv = O.profile_loglik(np.array([[0.1, 0.1], [0.9, 0.9]]), np.array([3.0, 4.0]), 1e-3, 0.5,
                          16, "dp", 1)
    assert pv[2] == 25.0 and pv[3] == 12.5


def test_oracle_special_functions():
    g = load_golden("bessel")
    for a, nu in enumerate(g["nus"]):
        got = O.bessel_k(float(nu), g["xs"])
        np.testing.assert_array_equal(got, g["vals"][a])
    for key in g:
        if key.startswith("matern_"):
            nu = float(key.split("_")[1])
            np.testing.assert_array_equal(O.matern(g["r"], 1.7, 0.13, nu), g[key])
    gam = np.array([O.gamma(float(x)) for x in g["gam_x"]])
    np.testing.assert_array_equal(gam, g["gam"])
    # frozen values of test_covmath.py:57-69,128-136
    assert O.bessel_k(0.5, np.array([1.0]))[0] == pytest.approx(0.46106850444789454, rel=1e-12)
    assert O.bessel_k(1.5, np.array([0.6]))[0] == pytest.approx(2.367970875005001, rel=1e-12)
    assert O.bessel_k(1.0, np.array([2.0]))[0] == pytest.approx(0.1398658818165224, rel=1e-10)
    assert O.matern(0.3, 2.0, 0.5, 1.5) == pytest.approx(1.7561972355008846, rel=1e-10)


def test_oracle_assembly_matches_reference():
    g = load_golden("assembly")
    for metric, mname, rng in (("euc", "euclidean", 0.2), ("gc", "great_circle", 900.0)):
        locs = g[f"{metric}_locs"]
        n = len(locs)
        for nu in (0.5, 1.0, 1.5, 0.35):
            for tag in ("dp", "mp2", "dst2"):
                mode = tag[:-1] if tag != "dp" else "dp"
                p = -(-n // 8)
                t = p if mode == "dp" else 2
                tiles = O.assemble(locs, (1.3, rng, nu), 8, mode, t, mname)
                dense = np.zeros((n, n))
                for (i, j), blk in tiles.items():
                    b = blk.astype(np.float64)
                    si = slice(8 * i, min(n, 8 * i + 8))
                    sj = slice(8 * j, min(n, 8 * j + 8))
                    if i == j:
                        dense[si, sj] = np.tril(b) + np.tril(b, -1).T
                    else:
                        dense[si, sj] = b
                        dense[sj, si] = b.T
                np.testing.assert_array_equal(dense, g[f"{metric}_{nu}_{tag}"])


def test_oracle_factor_small():
    g = load_golden("factor_small")
    n, nb = len(g["z"]), int(g["nb"])
    p = -(-n // nb)
    for tag, meta in g["results"].items():
        mode, t = tag_to_mode(tag, p)
        fac = O.cholesky(O.assemble(g["locs"], tuple(g["theta"]), nb, mode, t), n, nb, mode, t)
        key = tag.replace(":", "")
        low = np.zeros((n, n))
        for (i, j), (dp, sp) in fac.items():
            low[8 * i:8 * i + dp.shape[0], 8 * j:8 * j + dp.shape[1]] = np.tril(dp) if i == j else dp
        np.testing.assert_array_equal(low, g[f"lower_{key}"])
        assert O.logdet(fac, p) == meta["logdet"]
        np.testing.assert_array_equal(O.solve(fac, n, nb, g["z"]), g[f"solve_{key}"])
        assert list(O.planned_flops(n, nb, mode, t)) == pytest.approx(meta["flops"], rel=1e-12)


def test_oracle_flops_match_reference():
    with open(os.path.join(GOLDEN, "flops.json")) as fh:
        rows = json.load(fh)
    for n, nb, tag, fdp, fsp in rows:
        if n > 5000:
            continue  # O(p^3) loop; covered by the closed form in test_host
        p = -(-n // nb)
        mode, t = tag_to_mode(tag, p)
        got = O.planned_flops(n, nb, mode, t)
        assert got == pytest.approx((fdp, fsp), rel=1e-12), (n, nb, tag)
