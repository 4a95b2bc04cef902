"""Drop-in installation into the reference package `mixtile`.

The reference binds its hot-path functions by `from ... import ...` at import
time (mle.py:23-26, predict.py:13-17), so replacing `mixtile.factor.cholesky`
alone would not reroute `mixtile.loglik` or `mixtile.fit_matern`.  `install()`
rebinds every consumer's name to this library and makes the library raise the
reference's own exception classes, so existing callers (including the
reference's `loglik`, `profile_loglik`, `fit_matern`, `krige`,
`generate_field`) run on the GPU unchanged.  `uninstall()` restores the
originals.
"""

import importlib

_SAVED = []


def _targets(pkg):
    from . import factor as F
    from . import tilestore as T
    mod = lambda name: importlib.import_module(f"{pkg.__name__}.{name}")  # noqa: E731
    t, f, m = mod("tilestore"), mod("factor"), mod("mle")
    out = [
        (t, {"TileAssembler": T.TileAssembler, "assemble_covariance": T.assemble_covariance,
             "TileMatrix": T.TileMatrix}),
        (f, {"cholesky": F.cholesky, "logdet": F.logdet, "solve": F.solve,
             "matvec_lower": F.matvec_lower}),
        (m, {"TileAssembler": T.TileAssembler, "cholesky": F.cholesky,
             "factor_logdet": F.logdet, "factor_solve": F.solve}),
        (pkg, {"TileAssembler": T.TileAssembler, "assemble_covariance": T.assemble_covariance,
               "TileMatrix": T.TileMatrix, "cholesky": F.cholesky, "logdet": F.logdet, "solve": F.solve,
               "matvec_lower": F.matvec_lower}),
    ]
    from . import predict as P
    for opt in ("predict",):
        try:
            pm = mod(opt)
        except ImportError:
            continue
        # krige on the device (fused cross-covariance product); the reference's
        # own pmse_kfold looks krige up in its module, so it follows
        out.append((pm, {"cholesky": F.cholesky, "solve": F.solve,
                         "assemble_covariance": T.assemble_covariance, "krige": P.krige}))
    out.append((pkg, {"krige": P.krige}))
    # the reference CLI (cli.py:21-42) binds its own names: `mixtile bench`,
    # `estimate` and `predict` then run on the device too (cmd_bench,
    # cli.py:225-271: assemble -> cholesky -> logdet -> solve, residual vs DP)
    try:
        cm = mod("cli")
    except ImportError:
        cm = None
    if cm is not None:
        out.append((cm, {"TileAssembler": T.TileAssembler, "cholesky": F.cholesky,
                         "factor_logdet": F.logdet, "factor_solve": F.solve,
                         "reconstruction_error": F.reconstruction_error}))
    return out, f, t


def install(pkg=None):
    """Route `pkg` (default: the importable `mixtile`) through this library.

    Returns the list of (module, name) pairs that were rebound.
    """
    from . import factor as F
    from . import mle as M
    from . import tilestore as T
    pkg = pkg or importlib.import_module("mixtile")
    targets, ref_factor, ref_tilestore = _targets(pkg)
    # raise the reference's exception types from the GPU path
    for owner, name, new in ((F, "FactorizationError", ref_factor.FactorizationError),
                             (M, "FactorizationError", ref_factor.FactorizationError),
                             (T, "PrecisionOverflowError", ref_tilestore.PrecisionOverflowError),
                             (M, "PrecisionOverflowError", ref_tilestore.PrecisionOverflowError)):
        _SAVED.append((owner, name, getattr(owner, name)))
        setattr(owner, name, new)
    rebound = []
    for module, names in targets:
        for name, fn in names.items():
            if hasattr(module, name):
                _SAVED.append((module, name, getattr(module, name)))
                setattr(module, name, fn)
                rebound.append((module.__name__, name))
    return rebound


def uninstall():
    """Restore every name `install()` replaced."""
    while _SAVED:
        owner, name, old = _SAVED.pop()
        setattr(owner, name, old)
