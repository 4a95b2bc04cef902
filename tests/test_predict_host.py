"""CPU: kriging oracle and k-fold bookkeeping pinned to the reference.

tests/golden/krige.npz holds the reference's own predict.krige /
pmse_kfold / kfold_split outputs (tests/golden/make_golden.py).  The oracle
restatement of krige uses the same BLAS/LAPACK calls; `pmse_kfold` with a
custom predictor and `kfold_split` are pure host logic of this package and
need no GPU (predict.py:52-92, geodata.py:124-146).
"""

import math

import numpy as np
import pytest

from conftest import load_golden
from oracle import mixtile_oracle as O


@pytest.mark.parametrize("tag,mode,t", [("dp", "dp", 5), ("mp_1", "mp", 1), ("mp_2", "mp", 2)])
def test_oracle_krige_vs_reference(tag, mode, t):
    g = load_golden("krige")
    p = -(-len(g["z"]) // 64)
    pred = O.krige(g["locs"], g["z"], g["test"], tuple(g["theta"]), 64, mode,
                   p if mode == "dp" else t)
    np.testing.assert_allclose(pred, g[f"pred_{tag}"], rtol=0, atol=1e-12)


def test_kfold_split_matches_reference():
    import paper_2003_05324_b200 as mt
    g = load_golden("krige")
    f = mt.kfold_split(23, 4, seed=7)
    assert np.array_equal(f.fold_of, g["fold_of_23_4_7"])
    assert f.k == 4 and f.n == 23
    sizes = sorted(len(x) for x in f.folds)
    assert sizes == [5, 6, 6, 6]
    assert np.array_equal(np.sort(np.concatenate(f.folds)), np.arange(23))
    with pytest.raises(ValueError):
        mt.kfold_split(5, 1)
    with pytest.raises(ValueError):
        mt.kfold_split(3, 4)


def _ds(n, seed):
    import paper_2003_05324_b200 as mt
    rng = np.random.default_rng(seed)
    return mt.GeoDataset(mt.generate_locations(n, seed=seed), rng.standard_normal(n))


def test_pmse_truth_predictor_scores_zero():
    import paper_2003_05324_b200 as mt
    ds = _ds(30, 8)
    truth = {tuple(loc): val for loc, val in zip(ds.locations, ds.z)}
    rep = mt.pmse_kfold(ds, mt.MaternParams(1, .1, .5), 8, mt.PrecisionPolicy.dp(), k=5,
                        predictor=lambda tr, tl, th, pol: np.array([truth[tuple(x)] for x in tl]))
    assert rep.pmse == 0.0 and all(m == 0.0 for m in rep.fold_mse)
    assert np.array_equal(rep.predictions, ds.z)
    assert rep.as_dict()["k"] == 5


def test_pmse_zero_predictor_scores_signal_power():
    import paper_2003_05324_b200 as mt
    ds = _ds(23, 9)
    rep = mt.pmse_kfold(ds, mt.MaternParams(1, .1, .5), 8, mt.PrecisionPolicy.dp(), k=4,
                        predictor=lambda tr, tl, th, pol: np.zeros(len(tl)))
    assert math.isclose(rep.pmse, float(np.mean(ds.z ** 2)), rel_tol=1e-12)
    total = sum(m * len(f) for m, f in zip(rep.fold_mse, mt.kfold_split(23, 4, seed=0).folds))
    assert math.isclose(total / 23, rep.pmse, rel_tol=1e-12)


def test_pmse_rejects_bad_predictor_shape():
    import paper_2003_05324_b200 as mt
    ds = _ds(12, 14)
    with pytest.raises(ValueError):
        mt.pmse_kfold(ds, mt.MaternParams(1, .1, .5), 8, mt.PrecisionPolicy.dp(), k=3,
                      predictor=lambda tr, tl, th, pol: np.zeros(len(tl) + 1))


def test_krige_rejects_bad_test_shape_before_device():
    import paper_2003_05324_b200 as mt
    with pytest.raises(ValueError):
        mt.krige(_ds(10, 7), np.ones((3, 3)), mt.MaternParams(1, .1, .5), 8,
                 mt.PrecisionPolicy.dp())
    with pytest.raises(ValueError):
        mt.krige(_ds(10, 7), np.array([[np.nan, 0.0]]), mt.MaternParams(1, .1, .5), 8,
                 mt.PrecisionPolicy.dp())
