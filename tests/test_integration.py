"""CPU: install() rebinds the reference package's hot-path names (no compute).

Runs only where the reference package is importable (this build container);
the GPU box has no reference tree, so this test skips there."""

import importlib
import sys

import pytest

REF = "/root/reference/pkg/src"


@pytest.fixture
def mixtile():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    try:
        return importlib.import_module("mixtile")
    except ImportError:
        pytest.skip("reference package not importable here")


def test_install_rebinds_consumers(mixtile):
    import paper_2003_05324_b200 as mt
    from paper_2003_05324_b200 import factor as F
    from paper_2003_05324_b200 import integration
    orig = mixtile.mle.cholesky
    rebound = integration.install(mixtile)
    try:
        assert mixtile.mle.cholesky is mt.cholesky
        assert mixtile.mle.factor_solve is mt.solve and mixtile.mle.factor_logdet is mt.logdet
        assert mixtile.mle.TileAssembler is mt.TileAssembler
        assert mixtile.tilestore.assemble_covariance is mt.assemble_covariance
        assert mixtile.predict.cholesky is mt.cholesky
        assert mixtile.predict.krige is mt.krige
        # the reference CLI's bench/estimate/predict commands follow
        assert mixtile.cli.cholesky is mt.cholesky and mixtile.cli.TileAssembler is mt.TileAssembler
        assert mixtile.cli.factor_logdet is mt.logdet and mixtile.cli.factor_solve is mt.solve
        # the GPU path raises the reference's exception types
        assert F.FactorizationError is mixtile.factor.FactorizationError
        assert ("mixtile.mle", "cholesky") in rebound
    finally:
        integration.uninstall()
    assert mixtile.mle.cholesky is orig
    assert F.FactorizationError is not mixtile.factor.FactorizationError
