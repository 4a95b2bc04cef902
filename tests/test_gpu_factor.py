"""GPU: band-precision tile Cholesky, logdet and solves vs the reference.

Mirrors the reference's test_factor.py / test_kernels.py assertions on the
device path (csrc/potrf.cu, trsm.cu, update.cu, solve.cu via mt_cholesky,
mt_logdet, mt_solve), with the oracle / golden factors as the checker.
"""

import math

import numpy as np
import pytest

from conftest import load_golden, tag_to_mode
from oracle import mixtile_oracle as O

pytestmark = pytest.mark.gpu

THETA = (1.0, 0.1, 0.5)


def _mt():
    import paper_2003_05324_b200 as mt
    return mt


def _policy(mt, tag, p=None):
    if tag == "dp":
        return mt.PrecisionPolicy.dp()
    mode, t = tag.split(":")
    return (mt.PrecisionPolicy.mp(diag_thick=int(t)) if mode == "mp"
            else mt.PrecisionPolicy.dst(diag_thick=int(t)))


def _dataset(mt, n, seed=0):
    locs = mt.generate_locations(n, seed=seed)
    z = np.random.default_rng(seed + 1).standard_normal(n)
    return mt.GeoDataset(locs, z)


def _assemble(mt, n, nb, policy, seed=0, theta=THETA):
    return mt.assemble_covariance(_dataset(mt, n, seed), mt.MaternParams(*theta), nb, policy)


def _dense_cov(mt, n, seed=0, theta=THETA):
    locs = _dataset(mt, n, seed).locations
    return O.matern(O.pairwise(locs, locs), *theta)


def _lower(f):
    out = np.zeros((f.n, f.n))
    for (i, j), t in f.tiles.items():
        out[f.slice_of(i), f.slice_of(j)] = np.tril(t.dp) if i == j else t.dp
    return out


def _bitwise_equal(fa, fb):
    if fa.p != fb.p or set(fa.tiles) != set(fb.tiles):
        return False
    return all(fa.tiles[k].dp.tobytes() == fb.tiles[k].dp.tobytes() for k in fa.tiles)


# ------------------------------------------------------------------ dp path
@pytest.mark.parametrize("n,nb", [(32, 8), (6, 16), (37, 8), (300, 32), (1000, 128), (768, 256)])
def test_dp_factor_matches_dense(gpu, n, nb):
    mt = _mt()
    f = mt.cholesky(_assemble(mt, n, nb, mt.PrecisionPolicy.dp()))
    ref = np.linalg.cholesky(_dense_cov(mt, n))
    assert np.allclose(_lower(f), ref, rtol=0, atol=1e-11)


def test_golden_factors_all_policies(gpu):
    mt = _mt()
    g = load_golden("factor_small")
    n, nb = len(g["z"]), int(g["nb"])
    ds = mt.GeoDataset(g["locs"], g["z"])
    for tag, meta in g["results"].items():
        key = tag.replace(":", "")
        f = mt.cholesky(mt.assemble_covariance(ds, mt.MaternParams(*g["theta"]), nb,
                                               _policy(mt, tag)))
        low = _lower(f)
        ref = g[f"lower_{key}"]
        tol = 1e-12 if tag in ("dp", "mp:9", "dst:2") else 5e-6
        np.testing.assert_allclose(low, ref, rtol=0, atol=tol, err_msg=tag)
        assert math.isclose(mt.logdet(f), meta["logdet"], rel_tol=1e-12 if tol < 1e-9 else 1e-6)
        np.testing.assert_allclose(mt.solve(f, g["z"]), g[f"solve_{key}"],
                                   rtol=1e-9 if tol < 1e-9 else 1e-3, atol=1e-9)
        spmask = g[f"spmask_{key}"]
        for (i, j), t in f.tiles.items():
            assert (t.sp is not None) == bool(spmask[i, j]), (tag, i, j)
        assert f.flops.dp == pytest.approx(meta["flops"][0], rel=1e-12)
        assert f.flops.sp == pytest.approx(meta["flops"][1], rel=1e-12)


def test_identity_and_npd_index(gpu):
    mt = _mt()
    f = mt.cholesky(mt.TileMatrix.from_dense(np.eye(10), 4, mt.PrecisionPolicy.dp()))
    assert np.array_equal(_lower(f), np.eye(10)) and mt.logdet(f) == 0.0
    assert np.array_equal(mt.solve(f, np.arange(10.0)), np.arange(10.0))
    a = np.eye(48)
    a[37, 37] = -1.0
    with pytest.raises(mt.FactorizationError) as exc:
        mt.cholesky(mt.TileMatrix.from_dense(a, 8, mt.PrecisionPolicy.dp()))
    assert exc.value.index == 37
    # kernel-level hand values (test_kernels.py:24-44) on a single 2x2 tile
    f = mt.cholesky(mt.TileMatrix.from_dense(np.array([[4.0, 2.0], [2.0, 3.0]]), 2,
                                             mt.PrecisionPolicy.dp()))
    l = f.tiles[(0, 0)].dp
    assert l[0, 0] == 2.0 and l[1, 0] == 1.0 and abs(l[1, 1] - math.sqrt(2.0)) < 1e-15
    assert l[0, 1] == 2.0  # strict upper untouched
    with pytest.raises(mt.FactorizationError) as exc:
        mt.cholesky(mt.TileMatrix.from_dense(np.array([[1.0, 2.0], [2.0, 1.0]]), 2,
                                             mt.PrecisionPolicy.dp()))
    assert exc.value.index == 1


# --------------------------------------------------------------- mixed band
def test_mp_full_band_is_bitwise_dp(gpu):
    mt = _mt()
    f_dp = mt.cholesky(_assemble(mt, 30, 8, mt.PrecisionPolicy.dp()))
    f_mp = mt.cholesky(_assemble(mt, 30, 8, mt.PrecisionPolicy.mp(diag_thick=4)))
    assert f_mp.p == 4 and _bitwise_equal(f_dp, f_mp)
    assert all(t.sp is None for t in f_mp.tiles.values())
    big_dp = mt.cholesky(_assemble(mt, 1024, 128, mt.PrecisionPolicy.dp()))
    big_mp = mt.cholesky(_assemble(mt, 1024, 128, mt.PrecisionPolicy.mp(diag_thick=8)))
    assert _bitwise_equal(big_dp, big_mp)


def test_mp_matches_oracle_at_same_band(gpu):
    mt = _mt()
    for n, nb, t in ((64, 8, 1), (64, 8, 2), (1024, 128, 2), (1024, 256, 1)):
        ds = _dataset(mt, n)
        f = mt.cholesky(mt.assemble_covariance(ds, mt.MaternParams(*THETA), nb,
                                               mt.PrecisionPolicy.mp(diag_thick=t)))
        ref = O.cholesky(O.assemble(ds.locations, THETA, nb, "mp", t), n, nb, "mp", t)
        for key, (dp, sp) in ref.items():
            got = f.tiles[key]
            assert (got.sp is None) == (sp is None), key
            np.testing.assert_allclose(got.dp, dp, rtol=0, atol=5e-5, err_msg=str(key))
        # MP logdet: FP32-noise level, judged at the north-star MP tolerance
        assert math.isclose(mt.logdet(f), O.logdet(ref, f.p), rel_tol=1e-5)


def test_mp_residual_and_band_accuracy(gpu):
    mt = _mt()
    n = 64
    a = _dense_cov(mt, n)
    f_dp = mt.cholesky(_assemble(mt, n, 8, mt.PrecisionPolicy.dp()))
    f_mp = mt.cholesky(_assemble(mt, n, 8, mt.PrecisionPolicy.mp(diag_thick=1)))
    ref = _assemble(mt, n, 8, mt.PrecisionPolicy.dp())
    r_dp = mt.reconstruction_error(f_dp, ref)
    r_mp = mt.reconstruction_error(f_mp, ref)
    assert r_dp <= 1e-13 * n and r_mp <= 1e-5 * n and r_mp > r_dp
    f2 = mt.cholesky(_assemble(mt, n, 8, mt.PrecisionPolicy.mp(diag_thick=2)))
    low = _lower(f2)
    resid = a - low @ low.T
    for i in range(f2.p):
        for j in range(i + 1):
            nrm = np.linalg.norm(resid[f2.slice_of(i), f2.slice_of(j)])
            assert nrm <= (1e-13 if i - j < 2 else 1e-5) * n, (i, j, nrm)


def test_mp_off_band_payloads_are_fp32(gpu):
    mt = _mt()
    f = mt.cholesky(_assemble(mt, 40, 8, mt.PrecisionPolicy.mp(diag_thick=1)))
    for (i, j), t in f.tiles.items():
        assert t.dp is not None and t.dp.dtype == np.float64
        if i != j:
            assert t.sp is not None and t.sp.dtype == np.float32
            assert np.array_equal(t.dp, t.sp.astype(np.float64))


def test_schedule_invariance_bitwise(gpu):
    # lookahead 0 (single stream) vs 1 (panel stream): identical bits, any threads
    mt = _mt()
    for pol in (mt.PrecisionPolicy.mp(diag_thick=1), mt.PrecisionPolicy.mp(diag_thick=3),
                mt.PrecisionPolicy.dp()):
        outs = [mt.cholesky(_assemble(mt, 1536, 128, pol), threads=th, lookahead=la)
                for th, la in ((1, 0), (4, 1), (8, 1))]
        assert _bitwise_equal(outs[0], outs[1]) and _bitwise_equal(outs[0], outs[2])
        assert mt.logdet(outs[0]) == mt.logdet(outs[1]) == mt.logdet(outs[2])


# ---------------------------------------------------------------- sparsified
def test_dst_modes(gpu):
    mt = _mt()
    n, nb = 24, 4
    a = _dense_cov(mt, n)
    f = mt.cholesky(_assemble(mt, n, nb, mt.PrecisionPolicy.dst(diag_thick=1)))
    assert set(f.tiles) == {(k, k) for k in range(6)}
    for k in range(6):
        s = f.slice_of(k)
        assert np.allclose(np.tril(f.tiles[(k, k)].dp), np.linalg.cholesky(a[s, s]), atol=1e-13)
    rng = np.random.default_rng(3)
    l0 = np.zeros((n, n))
    for i in range(6):
        si = slice(i * nb, (i + 1) * nb)
        l0[si, si] = np.tril(rng.standard_normal((nb, nb))) + 4.0 * np.eye(nb)
        if i > 0:
            l0[si, slice((i - 1) * nb, i * nb)] = rng.standard_normal((nb, nb))
    b = l0 @ l0.T
    f_dp = mt.cholesky(mt.TileMatrix.from_dense(b, nb, mt.PrecisionPolicy.dp()))
    f_dst = mt.cholesky(mt.TileMatrix.from_dense(b, nb, mt.PrecisionPolicy.dst(diag_thick=2)))
    for key, t in f_dst.tiles.items():
        assert np.array_equal(t.dp, f_dp.tiles[key].dp), key
    c = np.array([[1.0, 0.8, 0.9], [0.8, 1.0, 0.8], [0.9, 0.8, 1.0]])
    mt.cholesky(mt.TileMatrix.from_dense(c, 1, mt.PrecisionPolicy.dp()))
    with pytest.raises(mt.FactorizationError):
        mt.cholesky(mt.TileMatrix.from_dense(c, 1, mt.PrecisionPolicy.dst(diag_thick=2)))


# -------------------------------------------------------------------- solves
def test_solves_and_logdet_vs_dense(gpu):
    mt = _mt()
    n = 40
    a = _dense_cov(mt, n)
    z = np.random.default_rng(5).standard_normal(n)
    f = mt.cholesky(_assemble(mt, n, 8, mt.PrecisionPolicy.dp()))
    assert np.allclose(mt.solve(f, z), np.linalg.solve(a, z), rtol=0, atol=1e-9)
    rhs = np.random.default_rng(6).standard_normal((n, 3))
    out = mt.solve(f, rhs)
    assert out.shape == (n, 3)
    for c in range(3):
        assert np.allclose(out[:, c], mt.solve(f, rhs[:, c]), rtol=0, atol=1e-12)
    with pytest.raises(ValueError):
        mt.solve(f, np.ones(n + 1))
    assert math.isclose(mt.logdet(f), float(np.sum(np.log(np.linalg.eigvalsh(a)))), rel_tol=1e-8)
    v = np.random.default_rng(9).standard_normal(n)
    assert np.allclose(mt.matvec_lower(f, v), _lower(f) @ v, rtol=0, atol=1e-12)
    y = mt.forward_solve(f, z)
    assert math.isclose(float(y @ y), float(z @ mt.solve(f, z)), rel_tol=1e-10)


def test_large_tile_factor_vs_oracle(gpu):
    # config-2 tile size (nb = 512): DP factor, logdet and solve vs the oracle
    mt = _mt()
    n, nb = 2048, 512
    ds = _dataset(mt, n, seed=4)
    f = mt.cholesky(mt.assemble_covariance(ds, mt.MaternParams(*THETA), nb,
                                           mt.PrecisionPolicy.dp()))
    ref = O.cholesky(O.assemble(ds.locations, THETA, nb, "dp", 4), n, nb, "dp", 4)
    for key, (dp, _) in ref.items():
        np.testing.assert_allclose(f.tiles[key].dp, dp, rtol=0, atol=1e-11, err_msg=str(key))
    assert math.isclose(mt.logdet(f), O.logdet(ref, 4), rel_tol=1e-11)
    np.testing.assert_allclose(mt.solve(f, ds.z), O.solve(ref, n, nb, ds.z), rtol=1e-8, atol=1e-8)


@pytest.mark.parametrize("n,nb,t,la", [(3000, 256, 2, 1), (4096, 512, 8, 1), (1500, 256, 6, 0)])
def test_fused_forward_sweep_bitwise(gpu, n, nb, t, la):
    """mt_cholesky_quad (forward sweep fused into the factorization schedule)
    equals mt_cholesky followed by mt_quad bit for bit: same kernels per column,
    issued as soon as the column is final."""
    import ctypes
    import torch
    mt = _mt()
    from paper_2003_05324_b200 import _lib
    lib, st = _lib.load(), _lib.stream_handle()
    locs = mt.generate_locations(n, seed=41)
    ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.random.default_rng(42).standard_normal(n)))
    asm = mt.TileAssembler(ds, nb)
    pol = mt.PrecisionPolicy.mp(diag_thick=t)
    outs = []
    for fused in (0, 1):
        m = mt.TileMatrix(n, nb, pol)
        asm.generate_into(m, mt.MaternParams(1.0, 0.1, 0.5))
        d = ctypes.byref(m.desc)
        work = torch.zeros(lib.mt_work_doubles(d), dtype=torch.float64, device=m.device)
        out = torch.zeros(1, dtype=torch.float64, device=m.device)
        if fused:
            _lib.check(lib.mt_cholesky_quad(d, la, _lib.ptr(asm.d_z), _lib.ptr(work), _lib.ptr(out),
                                            st), "mt_cholesky_quad")
        else:
            _lib.check(lib.mt_cholesky(d, la, st), "mt_cholesky")
            _lib.check(lib.mt_quad(d, _lib.ptr(asm.d_z), _lib.ptr(work), _lib.ptr(out), st), "mt_quad")
        torch.cuda.synchronize()
        outs.append(float(out.item()))
    assert outs[0] == outs[1]


@pytest.mark.parametrize("n,nb,pol", [(4096, 512, "mp:2"), (3000, 256, "dp"), (2048, 64, "mp:3"),
                                      (1920, 128, "dst:2")])
def test_cluster_potrf_bitwise_equals_single_cta(gpu, n, nb, pol):
    """Option 14: POTRF on a cluster of nb/32 CTAs (tile in distributed shared
    memory) or as three small launches per 32-column block applies the
    single-CTA kernel's operations in the same order: the factor (including
    the FP32 narrowing and the 32x32 inverses feeding the TRSM) is bitwise
    identical; ragged last tile included."""
    import paper_2003_05324_b200 as mt
    from paper_2003_05324_b200 import _lib
    lib = _lib.load()
    locs = mt.generate_locations(n, seed=41)
    ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.zeros(n)))
    mode, _, t = pol.partition(":")
    policy = (mt.PrecisionPolicy.dp() if mode == "dp" else
              getattr(mt.PrecisionPolicy, mode)(diag_thick=int(t)))
    facs = []
    for flag in (0, 1, 2):
        old = lib.mt_set_option(14, flag)
        try:
            facs.append(mt.cholesky(mt.assemble_covariance(ds, mt.MaternParams(1.0, 0.1, 0.5), nb,
                                                           policy)))
        except mt.FactorizationError as exc:  # DST can be indefinite: same pivot on both
            facs.append(exc.index)
        finally:
            lib.mt_set_option(14, old)
    if not hasattr(facs[0], "tiles"):
        assert facs[0] == facs[1] == facs[2]
        return
    for other in facs[1:]:
        for key in facs[0].tiles:
            a, b = facs[0].tiles[key], other.tiles[key]
            assert np.array_equal(a.dp, b.dp), key
            assert (a.sp is None) == (b.sp is None) and (a.sp is None or np.array_equal(a.sp, b.sp))


def test_cluster_potrf_not_positive_definite_index(gpu):
    """The cluster POTRF reports the same global pivot as the reference."""
    import paper_2003_05324_b200 as mt
    from paper_2003_05324_b200 import _lib
    lib = _lib.load()
    n, nb = 1024, 256
    rng = np.random.default_rng(3)
    x = rng.standard_normal((n, n))
    a = x @ x.T / n + np.eye(n)
    a[600, 600] = -5.0
    for flag in (0, 1, 2):
        old = lib.mt_set_option(14, flag)
        try:
            with pytest.raises(mt.FactorizationError) as exc:
                mt.cholesky(mt.TileMatrix.from_dense(a, nb, mt.PrecisionPolicy.dp()))
            assert exc.value.index == 600
        finally:
            lib.mt_set_option(14, old)


@pytest.mark.parametrize("n,nb,pol", [(8192, 512, "mp:3"), (5000, 256, "mp:1"), (4096, 256, "dp"),
                                      (3000, 256, "dst:2")])
def test_lookahead_two_bitwise(gpu, n, nb, pol):
    """Lookahead depth 2 (panels k+1 and k+2 formed on the panel stream while
    the bulk update applies step k; three ring slots) only moves work between
    streams: factor, logdet and quad are bitwise equal to lookahead 0 and 1."""
    import paper_2003_05324_b200 as mt
    locs = mt.generate_locations(n, seed=43)
    ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.random.default_rng(44).standard_normal(n)))
    mode, _, t = pol.partition(":")
    policy = (mt.PrecisionPolicy.dp() if mode == "dp" else
              getattr(mt.PrecisionPolicy, mode)(diag_thick=int(t)))
    th = mt.MaternParams(1.0, 0.1, 0.5)
    asm = mt.TileAssembler(ds, nb)
    outs, facs = [], []
    for la in (0, 1, 2):
        try:
            outs.append(mt.Evaluator(asm, policy, lookahead=la)(th))
        except mt.FactorizationError as exc:
            outs.append(("npd", exc.index))
        m = mt.TileMatrix(n, nb, policy, panel_slots=3 if la == 2 else 2)
        asm.generate_into(m, th)
        try:
            facs.append(mt.cholesky(m, lookahead=la))  # the factor keeps its matrix alive
        except mt.FactorizationError as exc:
            facs.append(exc.index)
    assert outs[0] == outs[1] == outs[2], outs
    if isinstance(facs[0], int):
        assert facs[0] == facs[1] == facs[2]
        return
    for key in facs[0].tiles:
        a, b, c = facs[0].tiles[key], facs[1].tiles[key], facs[2].tiles[key]
        assert np.array_equal(a.dp, b.dp) and np.array_equal(a.dp, c.dp), key
