"""GPU: the reference package's own entry points, executed through
integration.install() -- the drop-in claim end to end.

The unmodified reference (`mixtile`, installed into baseline/_ref by
`pip install --target baseline/_ref`, or the source tree where it exists) is
imported, install() rebinds its hot-path names, and then the reference's
`loglik`, `cholesky(TileMatrix.from_dense(...))`, `fit_matern` and the
`mixtile bench` CLI run with reference-built objects (its GeoDataset,
MaternParams, PrecisionPolicy) -- and must launch this library's kernels and
return the reference's answers."""

import importlib
import io
import json
import math
import os
import sys

import numpy as np
import pytest

from conftest import ROOT, load_golden

pytestmark = pytest.mark.gpu

_CANDIDATES = [os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"]


@pytest.fixture(scope="module")
def ref(gpu):
    for path in _CANDIDATES:
        if os.path.isdir(os.path.join(path, "mixtile")):
            if path not in sys.path:
                sys.path.insert(0, path)
            break
    try:
        mixtile = importlib.import_module("mixtile")
    except ImportError:
        pytest.skip("reference package not installed (baseline/_ref)")
    from paper_2003_05324_b200 import integration
    integration.install(mixtile)
    yield mixtile
    integration.uninstall()


def _launches():
    from paper_2003_05324_b200 import _lib
    return int(_lib.load().mt_launch_count())


def test_reference_loglik_runs_on_the_gpu(ref):
    g = load_golden("config1")
    ds = ref.GeoDataset(g["locs"], g["z"])
    th = ref.MaternParams(*(float(v) for v in g["theta"]))
    for tag, tol in (("dp", 1e-8), ("mp:2", 1e-5), ("mp:8", 1e-5)):
        pol = ref.PrecisionPolicy.dp() if tag == "dp" else ref.PrecisionPolicy.mp(
            diag_thick=int(tag.split(":")[1]))
        l0 = _launches()
        ev = ref.loglik(ds, th, 256, pol)
        assert _launches() > l0, "the reference's loglik did not reach the CUDA library"
        want = g["results"][tag][0]
        assert abs(ev.value - want) <= tol * abs(want), (tag, ev.value, want)
        assert type(ev).__module__.startswith("paper_2003_05324_b200") or hasattr(ev, "quad")


def test_reference_cholesky_of_from_dense(ref):
    """The reference test_factor.py pattern: cholesky(TileMatrix.from_dense(a, nb, pol))."""
    rng = np.random.default_rng(0)
    n, nb = 600, 128
    x = rng.standard_normal((n, n))
    a = x @ x.T / n + np.eye(n)
    want = np.linalg.cholesky(a)
    for pol in (ref.PrecisionPolicy.dp(), ref.PrecisionPolicy.mp(diag_thick=2)):
        fac = ref.cholesky(ref.TileMatrix.from_dense(a, nb, pol))
        low = np.zeros((n, n))
        for (i, j), t in fac.tiles.items():
            blk = t.dp
            low[fac.slice_of(i), fac.slice_of(j)] = np.tril(blk) if i == j else blk
        tol = 1e-10 if pol.mode.value == "dp" else 1e-4
        assert np.max(np.abs(low - want)) <= tol
        assert math.isclose(ref.logdet(fac), 2 * np.sum(np.log(np.diag(want))), rel_tol=1e-6)


def test_reference_host_tilematrix_factored_in_place(ref):
    """A TileMatrix the reference itself built (host tile dict) is uploaded,
    factored on the GPU and overwritten in place (factor.py:238, 285)."""
    from mixtile import tilestore as T0
    host_cls = [c for c in T0.__dict__.values() if isinstance(c, type) and c.__name__ == "TileMatrix"]
    import paper_2003_05324_b200.integration as integ
    orig = next((old for owner, name, old in integ._SAVED
                 if name == "TileMatrix" and owner is T0), None)
    assert orig is not None and host_cls
    rng = np.random.default_rng(1)
    n, nb = 500, 96
    x = rng.standard_normal((n, n))
    a = x @ x.T / n + np.eye(n)
    m = orig.from_dense(a, nb, ref.PrecisionPolicy.dp())
    assert not hasattr(m, "desc")
    ref.cholesky(m)
    want = np.linalg.cholesky(a)
    for (i, j), t in m.tiles.items():
        blk = want[m.slice_of(i), m.slice_of(j)]
        got = np.tril(t.dp) if i == j else t.dp
        assert np.max(np.abs(got - blk)) <= 1e-10
    # a missing diagonal tile raises ValueError, as in the reference
    m2 = orig.from_dense(a, nb, ref.PrecisionPolicy.dp())
    del m2.tiles[(1, 1)]
    with pytest.raises(ValueError):
        ref.cholesky(m2)
    # not positive definite: the reference's own exception type and index
    b = a.copy()
    b[137, 137] = -1.0
    with pytest.raises(ref.FactorizationError) as exc:
        ref.cholesky(orig.from_dense(b, nb, ref.PrecisionPolicy.dp()))
    assert exc.value.index <= 137


def test_reference_fit_matern_through_install(ref):
    g = load_golden("fit_small")
    ds = ref.GeoDataset(g["locs"], g["z"])
    for tag, meta in g["results"].items():
        pol = ref.PrecisionPolicy.dp() if tag == "dp" else ref.PrecisionPolicy.mp(
            diag_thick=int(tag.split(":")[1]))
        l0 = _launches()
        fit = ref.fit_matern(ds, 32, pol)
        assert _launches() > l0
        for got, want in zip(fit.params.as_tuple(), meta["params"]):
            assert abs(got - want) <= 5e-4 * abs(want), (tag, got, want)


def test_reference_bench_cli_runs_on_the_gpu(ref):
    out = io.StringIO()
    l0 = _launches()
    from mixtile import cli
    old = sys.stdout
    sys.stdout = out
    try:
        rc = cli.main(["bench", "--n", "2048", "--nb", "256", "--policy", "dp", "--policy", "mp:2",
                       "--reps", "1", "--seed", "0"])
    finally:
        sys.stdout = old
    assert rc in (0, None)
    assert _launches() > l0
    rows = [ln for ln in out.getvalue().splitlines() if ln and not ln.startswith("#")]
    assert rows[0].startswith("n,nb,policy")
    body = [r.split(",") for r in rows[1:]]
    assert [r[2] for r in body] == ["dp", "mp:t2"] or len(body) == 2
    resid = [float(r[6]) for r in body]
    assert resid[0] < 1e-9 and resid[1] < 1e-3
