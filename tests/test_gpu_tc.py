"""GPU: the tcgen05 3xTF32 off-band update vs the SIMT FFMA update and the
reference.  3xTF32 is only acceptable if it matches FP32 accuracy
(north_star): both engines must sit within the MP tolerance of the CPU
reference at the same band, and 3xTF32's distance to the reference must be
within a small factor of FFMA's."""

import math

import numpy as np
import pytest

from conftest import load_golden
from oracle import mixtile_oracle as O

pytestmark = pytest.mark.gpu


def _mt():
    import paper_2003_05324_b200 as mt
    return mt


@pytest.fixture
def rz_engine(gpu):
    """The opt-in whole-K TMEM engine: its kernel variants (single CTA, CTA
    pairs, 256 x 512 items) apply identical MMA sequences and must agree bitwise."""
    mt = _mt()
    old = mt.set_fp32_engine("tf32x3_rz")
    yield mt
    mt.set_fp32_engine(old)


@pytest.fixture
def engine(gpu):
    mt = _mt()
    old = mt.set_fp32_engine("tf32x3")
    yield mt
    mt.set_fp32_engine(old)


def _factor(mt, ds, theta, nb, t, eng, lookahead=1):
    mt.set_fp32_engine(eng)
    return mt.cholesky(mt.assemble_covariance(ds, mt.MaternParams(*theta), nb,
                                              mt.PrecisionPolicy.mp(diag_thick=t)),
                       lookahead=lookahead)


def test_tf32x3_factor_accuracy_vs_ffma_and_oracle(engine):
    mt = engine
    n, nb, t = 2048, 256, 2
    theta = (1.0, 0.1, 0.5)
    locs = mt.generate_locations(n, seed=3)
    ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.zeros(n)))
    ref = O.cholesky(O.assemble(ds.locations, theta, nb, "mp", t), n, nb, "mp", t)
    f_tc = _factor(mt, ds, theta, nb, t, "tf32x3")
    f_ff = _factor(mt, ds, theta, nb, t, "ffma")
    err_tc = err_ff = 0.0
    for key, (dp, _) in ref.items():
        err_tc = max(err_tc, float(np.max(np.abs(f_tc.tiles[key].dp - dp))))
        err_ff = max(err_ff, float(np.max(np.abs(f_ff.tiles[key].dp - dp))))
    assert err_ff < 5e-5 and err_tc < 5e-5, (err_tc, err_ff)
    # FP32 accuracy gate (north_star: 3xTF32 only if it matches FP32): the
    # default engine restarts the TMEM accumulation every 32 K-columns and sums
    # the chunks with round-to-nearest (tcf_update.cu); measured on B200 at
    # 0.27x the round-to-nearest FFMA engine's distance from the reference factor
    assert err_tc <= 1.5 * err_ff, (err_tc, err_ff)
    # band tiles of rows k < t are untouched by FP32 work: equal across engines
    assert np.array_equal(f_tc.tiles[(0, 0)].dp, f_ff.tiles[(0, 0)].dp)


def test_tf32x3_loglik_config1_parity(engine):
    mt = engine
    g = load_golden("config1")
    ds = mt.GeoDataset(g["locs"], g["z"])
    theta = mt.MaternParams(*g["theta"])
    for tag in ("mp:1", "mp:2", "mp:4", "mp:8"):
        t = int(tag.split(":")[1])
        want = g["results"][tag][0]
        mt.set_fp32_engine("tf32x3")
        a = mt.loglik(ds, theta, 256, mt.PrecisionPolicy.mp(diag_thick=t))
        mt.set_fp32_engine("ffma")
        b = mt.loglik(ds, theta, 256, mt.PrecisionPolicy.mp(diag_thick=t))
        ra = abs(a.value - want) / abs(want)
        rb = abs(b.value - want) / abs(want)
        assert ra <= 1e-5 and rb <= 1e-5, (tag, ra, rb)


def test_tf32x3_deterministic_and_schedule_invariant(engine):
    mt = engine
    n, nb = 3072, 256
    locs = mt.generate_locations(n, seed=8)
    ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.zeros(n)))
    outs = [_factor(mt, ds, (1.0, 0.1, 0.5), nb, 1, "tf32x3", lookahead=la) for la in (1, 1, 0)]
    for key in outs[0].tiles:
        a = outs[0].tiles[key].dp.tobytes()
        assert a == outs[1].tiles[key].dp.tobytes() == outs[2].tiles[key].dp.tobytes(), key


def test_tf32x3_large_tile_512(engine):
    # config-2 tile size: nb = 512 exercises 4x2 work items per output tile
    mt = engine
    n, nb, t = 4096, 512, 2
    theta = (1.0, 0.1, 0.5)
    locs = mt.generate_locations(n, seed=11)
    z = np.random.default_rng(12).standard_normal(n)
    ds, _ = mt.morton_sort(mt.GeoDataset(locs, z))
    ev = mt.loglik(ds, mt.MaternParams(*theta), nb, mt.PrecisionPolicy.mp(diag_thick=t))
    want, _, _ = O.loglik(ds.locations, ds.z, theta, nb, "mp", t)
    assert abs(ev.value - want) / abs(want) <= 1e-5


@pytest.mark.parametrize("mode,t", [("dp", None), ("mp", 2), ("mp", 3)])
def test_tma_dmma_update_bitwise_equals_register_staged(gpu, mode, t):
    """The TMA-staged DMMA band update applies the same DMMA sequence per
    output element as the register-staged kernel: factors are bitwise equal."""
    mt = _mt()
    n, nb = 1920, 256  # ragged last tile row
    theta = (1.0, 0.1, 0.5)
    locs = mt.generate_locations(n, seed=5)
    ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.zeros(n)))
    pol = mt.PrecisionPolicy.dp() if mode == "dp" else mt.PrecisionPolicy.mp(diag_thick=t)
    facs = []
    for legacy in (0, 1):
        old = mt.set_legacy_dmma(legacy)
        try:
            facs.append(mt.cholesky(mt.assemble_covariance(ds, mt.MaternParams(*theta), nb, pol)))
        finally:
            mt.set_legacy_dmma(old)
    a, b = facs
    for key in a.tiles:
        ta, tb = a.tiles[key], b.tiles[key]
        if ta.dp is not None and tb.dp is not None and a.matrix.band(*key):
            assert np.array_equal(ta.dp, tb.dp), key


@pytest.mark.parametrize("n,nb,t", [(2048, 256, 2), (2000, 256, 1), (3072, 512, 2)])
def test_tc_trsm_matches_substitution_and_oracle(engine, n, nb, t):
    """Off-band TRSM as a 3xTF32 GEMM against L_kk^{-1}: FP32-class accuracy,
    within a small factor of the SIMT substitution, ragged last tile included."""
    mt = engine
    theta = (1.0, 0.1, 0.5)
    locs = mt.generate_locations(n, seed=11)
    ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.zeros(n)))
    ref = O.cholesky(O.assemble(ds.locations, theta, nb, "mp", t), n, nb, "mp", t)
    facs = {}
    for flag in (1, 0):
        old = mt.set_tc_trsm(flag)
        try:
            facs[flag] = _factor(mt, ds, theta, nb, t, "tf32x3")
        finally:
            mt.set_tc_trsm(old)
    errs = {}
    for flag, f in facs.items():
        e = 0.0
        for key, (dp, _) in ref.items():
            e = max(e, float(np.max(np.abs(f.tiles[key].dp - dp))))
        errs[flag] = e
    assert errs[1] < 5e-5 and errs[0] < 5e-5, errs
    assert errs[1] <= 8.0 * errs[0] + 1e-7, errs


def test_tc_trsm_loglik_parity_strong_field(engine):
    """Strong-correlation field (beta=0.3, nu=1): the ill-conditioned case for
    an inverse-based solve; the MP tolerance vs the reference must still hold."""
    mt = engine
    g = load_golden("strong1024")
    ds = mt.GeoDataset(g["locs"], g["z"])
    theta = tuple(float(v) for v in g["theta"])
    nb, t = 256, 1
    ref, _, _ = O.loglik(ds.locations, ds.z, theta, nb, "mp", t)
    dp = g["results"]["dp"][0]
    cpu_gap = abs(ref - dp) / abs(dp)  # the reference's own MP error on this field
    for flag in (1, 0):
        old = mt.set_tc_trsm(flag)
        try:
            ev = mt.loglik(ds, mt.MaternParams(*theta), nb, mt.PrecisionPolicy.mp(diag_thick=t))
        finally:
            mt.set_tc_trsm(old)
        gpu_gap = abs(ev.value - dp) / abs(dp)
        rel = abs(ev.value - ref) / abs(ref)
        print(f"strong1024 tc_trsm={flag}: GPU-MP vs CPU-MP {rel:.2e}; vs DP GPU {gpu_gap:.2e} "
              f"CPU {cpu_gap:.2e}")
        # the north-star MP tolerance, or -- on this ill-conditioned field, where
        # two FP32 factorizations differ by up to the method's own error -- no
        # further from DP than the reference's MP (1.5x rounding-noise margin)
        assert rel <= 1e-5 or gpu_gap <= 1.5 * cpu_gap, (flag, ev.value, ref, dp)


@pytest.mark.parametrize("ysms", [1, 32, 200])
def test_sm_yield_keeps_results_bitwise(gpu, ysms):
    """The bulk update's SM-yield protocol only changes which CTA runs which
    work item: factors equal the no-yield run bit for bit, including small
    launches where every running CTA could be asked to yield."""
    mt = _mt()
    from paper_2003_05324_b200 import _lib
    lib = _lib.load()
    n, nb, t = 4096, 256, 2
    locs = mt.generate_locations(n, seed=9)
    ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.zeros(n)))
    pol = mt.PrecisionPolicy.mp(diag_thick=t)
    facs = []
    for y in (0, ysms):
        old = lib.mt_set_option(5, y)
        try:
            facs.append(mt.cholesky(mt.assemble_covariance(ds, mt.MaternParams(1.0, 0.1, 0.5), nb,
                                                           pol), lookahead=1))
        finally:
            lib.mt_set_option(5, old)
    for key in facs[0].tiles:
        a, b = facs[0].tiles[key], facs[1].tiles[key]
        assert np.array_equal(a.dp, b.dp), key


@pytest.mark.parametrize("n,nb,t", [(8192, 512, 3), (6144, 256, 2)])
def test_coscheduled_band_update_bitwise(gpu, n, nb, t):
    """Option 10 (FP64 band update launched as a programmatic dependent beside a
    capped FP32 update) changes only where and when work runs: bitwise equal."""
    mt = _mt()
    from paper_2003_05324_b200 import _lib
    lib = _lib.load()
    locs = mt.generate_locations(n, seed=29)
    ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.zeros(n)))
    pol = mt.PrecisionPolicy.mp(diag_thick=t)
    facs = []
    for co in (0, 1):
        old = lib.mt_set_option(10, co)
        try:
            facs.append(mt.cholesky(mt.assemble_covariance(ds, mt.MaternParams(1.0, 0.1, 0.5), nb,
                                                           pol), lookahead=1))
        finally:
            lib.mt_set_option(10, old)
    for key in facs[0].tiles:
        assert np.array_equal(facs[0].tiles[key].dp, facs[1].tiles[key].dp), key


@pytest.mark.parametrize("n,t,co", [(8192, 3, 1), (7000, 2, 0), (12288, 8, 1)])
def test_wide_pair_items_bitwise(rz_engine, n, t, co):
    """Option 12 (bulk update on 256 x 512 CTA-pair items, single-buffered TMEM)
    applies the same MMA sequence per output element: bitwise equal to the
    256 x 256-item kernel, with and without co-scheduling, ragged last tile."""
    mt = _mt()
    from paper_2003_05324_b200 import _lib
    lib = _lib.load()
    locs = mt.generate_locations(n, seed=31)
    ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.zeros(n)))
    pol = mt.PrecisionPolicy.mp(diag_thick=t)
    facs = []
    oc = lib.mt_set_option(10, co)
    try:
        for wide in (0, 1):
            old = lib.mt_set_option(12, wide)
            try:
                facs.append(mt.cholesky(mt.assemble_covariance(ds, mt.MaternParams(1.0, 0.1, 0.5),
                                                               512, pol), lookahead=1))
            finally:
                lib.mt_set_option(12, old)
    finally:
        lib.mt_set_option(10, oc)
    for key in facs[0].tiles:
        assert np.array_equal(facs[0].tiles[key].dp, facs[1].tiles[key].dp), key


@pytest.mark.parametrize("n,t,co", [(8192, 3, 1), (7000, 2, 0), (12288, 8, 1)])
def test_tcf_four_cta_clusters_bitwise(gpu, n, t, co):
    """Option 15: the round-to-nearest engine on 4-CTA clusters (two CTA pairs
    on 512 x 256 items, the B operand multicast across the pairs) applies the
    same MMA / flush / FADD sequence per output element as the 2-CTA kernel:
    bitwise equal factors (bulk, panel-column update and TRSM), with and
    without co-scheduling, ragged last tile included."""
    mt = _mt()
    from paper_2003_05324_b200 import _lib
    lib = _lib.load()
    locs = mt.generate_locations(n, seed=37)
    ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.zeros(n)))
    pol = mt.PrecisionPolicy.mp(diag_thick=t)
    facs = []
    oc = lib.mt_set_option(10, co)
    try:
        for c4 in (0, 1):
            old = lib.mt_set_option(15, c4)
            try:
                facs.append(mt.cholesky(mt.assemble_covariance(ds, mt.MaternParams(1.0, 0.1, 0.5),
                                                               512, pol), lookahead=1))
            finally:
                lib.mt_set_option(15, old)
    finally:
        lib.mt_set_option(10, oc)
    for key in facs[0].tiles:
        assert np.array_equal(facs[0].tiles[key].dp, facs[1].tiles[key].dp), key


@pytest.mark.parametrize("n,t,co,c4", [(8192, 3, 1, 0), (7000, 2, 0, 0), (12288, 8, 1, 1)])
def test_tcf_reduce_add_bitwise(gpu, n, t, co, c4):
    """Option 17: the FP32 update writes -sum and lets the TMA unit add it into
    C at L2 (C + (-sum) == C - sum in IEEE arithmetic) instead of loading C
    into shared memory and storing C - sum: bitwise equal factors, panel-column
    updates with the fused TF32 split and ragged last tiles included."""
    mt = _mt()
    from paper_2003_05324_b200 import _lib
    lib = _lib.load()
    locs = mt.generate_locations(n, seed=41)
    ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.zeros(n)))
    pol = mt.PrecisionPolicy.mp(diag_thick=t)
    facs = []
    oc, o4 = lib.mt_set_option(10, co), lib.mt_set_option(15, c4)
    try:
        for red in (0, 1):
            old = lib.mt_set_option(17, red)
            try:
                facs.append(mt.cholesky(mt.assemble_covariance(ds, mt.MaternParams(1.0, 0.1, 0.5),
                                                               512, pol), lookahead=1))
            finally:
                lib.mt_set_option(17, old)
    finally:
        lib.mt_set_option(10, oc)
        lib.mt_set_option(15, o4)
    for key in facs[0].tiles:
        assert np.array_equal(facs[0].tiles[key].dp, facs[1].tiles[key].dp), key
