"""CPU: host logic of the drop-in (policy, flop plan, synthetic inputs) and the
C-ABI surface of libmixtile_b200.so (loads and exports every declared symbol;
no compute calls here)."""

import ctypes
import json
import math
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, load_golden, tag_to_mode

from paper_2003_05324_b200 import _lib
from paper_2003_05324_b200.factor import _plan_flops, planned_flops
from paper_2003_05324_b200.geodata import (
    GeoDataset, derive_seed, generate_locations, morton_sort)
from paper_2003_05324_b200.tilestore import (
    Mode, PrecisionPolicy, band_member, percent_to_thickness)


@pytest.mark.parametrize("pct,p,expect", [(10, 20, 2), (1, 20, 1), (100, 20, 20), (50, 7, 4),
                                          (100, 1, 1)])
def test_percent_to_thickness(pct, p, expect):
    assert percent_to_thickness(pct, p) == expect


@pytest.mark.parametrize("pct", [0, -5, 101])
def test_percent_to_thickness_rejects(pct):
    with pytest.raises(ValueError):
        percent_to_thickness(pct, 10)


def test_policy_resolution_and_band():
    assert PrecisionPolicy.mp(dp_percent=10).resolve(20).diag_thick == 2
    assert PrecisionPolicy.dp().resolve(7).diag_thick == 7
    for bad in (PrecisionPolicy.mp(diag_thick=0), PrecisionPolicy.mp(diag_thick=6),
                PrecisionPolicy.mp()):
        with pytest.raises(ValueError):
            bad.resolve(5)
    mp2 = PrecisionPolicy.mp(diag_thick=2).resolve(5)
    assert band_member(2, 1, mp2) and not band_member(3, 1, mp2)
    assert band_member(4, 0, PrecisionPolicy.dp().resolve(5))
    assert PrecisionPolicy.dst(diag_thick=2).label() == "dst:t2"
    assert PrecisionPolicy.mp(dp_percent=10).label() == "mp:10"


def test_planned_flops_match_reference_plan():
    with open(os.path.join(GOLDEN, "flops.json")) as fh:
        rows = json.load(fh)
    for n, nb, tag, fdp, fsp in rows:
        p = -(-n // nb)
        mode, t = tag_to_mode(tag, p)
        pol = (PrecisionPolicy.dp() if mode == "dp" else
               PrecisionPolicy.mp(diag_thick=t) if mode == "mp" else PrecisionPolicy.dst(diag_thick=t))
        got = planned_flops(n, nb, pol)
        assert got.dp == pytest.approx(fdp, rel=1e-12) and got.sp == pytest.approx(fsp, rel=1e-12)


def test_flop_total_and_closed_form():
    for pol in (PrecisionPolicy.dp(), PrecisionPolicy.mp(diag_thick=2)):
        assert math.isclose(planned_flops(64, 8, pol).total, 64 ** 3 / 3.0, rel_tol=1e-12)
    # closed form (p > 64) agrees with the task-by-task plan
    a = planned_flops(130 * 16, 16, PrecisionPolicy.mp(diag_thick=3))
    b = _plan_flops(130 * 16, 16, 130, Mode.MP, 3)
    assert a.dp == pytest.approx(b.dp, rel=1e-12) and a.sp == pytest.approx(b.sp, rel=1e-12)
    assert planned_flops(128, 8, PrecisionPolicy.mp(dp_percent=10)).sp_fraction >= 0.70


def test_synthetic_locations_match_reference():
    g = load_golden("config1")
    locs = generate_locations(4096, seed=derive_seed(0, 0))
    ds, _ = morton_sort(GeoDataset(locs, np.zeros(4096)))
    np.testing.assert_array_equal(ds.locations, g["locs"])


def test_dataset_validation():
    with pytest.raises(ValueError):
        GeoDataset(np.zeros((3, 3)), np.zeros(3))
    with pytest.raises(ValueError):
        GeoDataset(np.zeros((3, 2)), np.zeros(2))
    with pytest.raises(ValueError):
        GeoDataset(np.array([[0.0, np.nan]]), np.zeros(1))


def _declared_functions():
    hdr = open(os.path.join(ROOT, "include", "mixtile_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(mt_[a-z0-9_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()  # dlopen only; needs no GPU
    names = _declared_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} not bound in _lib.SIGNATURES"
    assert lib.mt_version() >= 10


def test_layout_sizes_without_gpu():
    lib = _lib.load()
    # config 2: p = 128 -> 8256 lower tiles; t = 2: 255 band + 8001 off-band
    assert lib.mt_dp_tiles(128, 2, 1) == 255
    assert lib.mt_sp_tiles(128, 2, 1) == 8001
    assert lib.mt_sp_tiles(128, 1, 1) == 8128
    assert lib.mt_dp_tiles(128, 128, 0) == 8256
    assert lib.mt_sp_tiles(128, 128, 0) == 0
    assert lib.mt_dp_tiles(512, 8, 1) == 4068
    assert lib.mt_sp_tiles(512, 8, 1) == 127260
    assert lib.mt_dp_tiles(6, 2, 2) == 11 and lib.mt_sp_tiles(6, 2, 2) == 0


def test_matern_constants_host():
    th = _lib.matern_struct(1.0, 0.3, 1.0)
    assert th.kind == 2 and th.nl == 1 and th.mu == 0.0
    assert th.gam1 == pytest.approx(-0.5772156649015329)
    th = _lib.matern_struct(1.0, 0.1, 0.5)
    assert th.kind == 0
    with pytest.raises(ValueError):
        _lib.matern_struct(-1.0, 0.1, 0.5)
