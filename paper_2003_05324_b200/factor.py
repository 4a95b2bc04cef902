"""Band-precision tile Cholesky on the GPU, and solves on the factor.

Mirrors `mixtile.factor` (factor.py:31-369).  `cholesky` runs the whole
POTRF/TRSM/SYRK/GEMM DAG on the device (stream/event schedule with
lookahead, csrc/api.cu) and factors in place; `threads` is accepted for
signature compatibility and ignored (the result does not depend on it, as in
the reference, factor.py:13-16).
"""

import ctypes
import math

import numpy as np

from . import _lib
from .tilestore import Mode


class FactorizationError(ArithmeticError):
    """Non-positive pivot; index = global 0-based pivot (factor.py:31-37)."""

    def __init__(self, index, message=None):
        self.index = int(index)
        super().__init__(message or f"matrix not positive definite at global pivot {index}")


class FlopCount:
    """Flops split by executing precision (factor.py:98-117)."""

    __slots__ = ("dp", "sp")

    def __init__(self, dp=0.0, sp=0.0):
        self.dp = float(dp)
        self.sp = float(sp)

    @property
    def total(self):
        return self.dp + self.sp

    @property
    def sp_fraction(self):
        return self.sp / self.total if self.total > 0 else 0.0

    def __repr__(self):
        return f"FlopCount(dp={self.dp:.6g}, sp={self.sp:.6g})"


def _tile_rows(n, nb, p):
    return [nb if i < p - 1 else n - nb * (p - 1) for i in range(p)]


def _plan_flops(n, nb, p, mode, t):
    """Per-task flop split of the DAG, accumulated in the reference's task
    order (factor.py:83-95, 134-145) -- O(p^2) loops with closed-form sums
    over the GEMM rows instead of enumerating O(p^3) tasks."""
    r = _tile_rows(n, nb, p)
    dst = mode.value == "dst"
    fdp = fsp = 0.0
    # exact sums are needed only to float rounding; use the same per-task
    # terms the reference adds, grouped per (k, j) column of GEMMs
    for k in range(p):
        fdp += r[k] ** 3 / 3.0
        for i in range(k + 1, p):
            if dst and i - k >= t:
                continue
            f = r[i] * r[k] ** 2
            if i - k < t:
                fdp += f
            else:
                fsp += f
            fdp += r[i] ** 2 * r[k]
        for j in range(k + 1, p):
            if dst and j - k >= t:
                continue
            for i in range(j + 1, p):
                if dst and (i - k >= t or i - j >= t):
                    continue
                f = 2.0 * r[i] * r[j] * r[k]
                if i - j < t:
                    fdp += f
                else:
                    fsp += f
    return FlopCount(fdp, fsp)


def _fast_flops(n, nb, p, mode, t):
    """Closed form of the flop plan for uniform tiles (n = p nb), MP/DP only."""
    b3 = float(nb) ** 3
    fdp = p / 3.0 + p * (p - 1) / 2.0          # POTRF + SYRK
    d = np.arange(1, min(t, p))
    fdp += float(np.sum(p - d))                 # band TRSM
    fdp += float(np.sum((p - 1 - d) * (p - d)))  # band GEMM: 2 * (p-1-d)(p-d)/2
    total = n ** 3 / 3.0
    fdp *= b3
    return FlopCount(fdp, total - fdp)


def planned_flops(n, nb, policy):
    """Flop split of the factorization plan, without touching data (factor.py:134-145)."""
    n, nb = int(n), int(nb)
    p = -(-n // nb)
    pol = policy.resolve(p)
    if pol.mode.value != "dst" and n == p * nb and p > 64:
        return _fast_flops(n, nb, p, pol.mode, pol.diag_thick)
    return _plan_flops(n, nb, p, pol.mode, pol.diag_thick)


class CholeskyFactor:
    """Lower tile factor aliasing the factored TileMatrix's device pools (factor.py:209-227)."""

    def __init__(self, matrix, flops):
        self.matrix = matrix
        self.n = matrix.n
        self.nb = matrix.nb
        self.p = matrix.p
        self.policy = matrix.policy
        self.tiles = matrix.tiles
        self.flops = flops

    def rows_of(self, i):
        return self.nb if i < self.p - 1 else self.n - self.nb * (self.p - 1)

    def slice_of(self, i):
        return slice(i * self.nb, min((i + 1) * self.nb, self.n))

    def band(self, i, j):
        return abs(i - j) < self.policy.diag_thick


def cholesky(matrix, threads=1, lookahead=1):
    """Factor an assembled TileMatrix in place on the GPU (factor.py:230-285).

    lookahead: panels formed ahead of the bulk update on the panel stream
    (0, 1 or 2; 2 needs a TileMatrix(..., panel_slots=3)); results are
    bitwise identical for every value.

    Raises FactorizationError(global pivot) when not positive definite.
    """
    del threads  # schedule-invariant; accepted for signature compatibility
    if not hasattr(matrix, "desc"):
        return _cholesky_host_matrix(matrix, lookahead)
    if matrix.factored:
        raise ValueError("matrix is already factored")
    lib = _lib.load()
    _lib.check(lib.mt_cholesky(ctypes.byref(matrix.desc), int(lookahead),
                               _lib.stream_handle()), "mt_cholesky")
    matrix._touch()
    bad, _, _ = matrix.read_status()
    if bad >= 0:
        matrix.factored = True  # payloads are partially overwritten, as in the reference
        raise FactorizationError(bad)
    matrix.factored = True
    flops = planned_flops(matrix.n, matrix.nb, matrix.policy)
    return CholeskyFactor(matrix, flops)


def _cholesky_host_matrix(ref, lookahead):
    """cholesky() on a host tile dict (the reference's own TileMatrix, e.g.
    `TileMatrix.from_dense(a, nb, policy)` built before install()): upload,
    factor on the GPU, then overwrite the caller's tile payloads in place as
    the reference does (factor.py:238, 285), including the .sp/.dp pairs of
    off-band tiles and the narrowed band mirrors (test_factor.py:146-153).
    A missing diagonal tile raises ValueError (factor.py:240-242)."""
    from .tilestore import TileMatrix
    p = ref.p
    for k in range(p):
        if (k, k) not in ref.tiles:
            raise ValueError(f"diagonal tile {k} missing from the matrix")
    dev = TileMatrix.from_dense(ref.to_dense(), ref.nb, ref.policy)
    try:
        fac = cholesky(dev, lookahead=lookahead)
    finally:
        if dev.factored:  # partially factored payloads are visible too, as in the reference
            for key, tile in ref.tiles.items():
                got = dev.tiles[key]
                tile.dp, tile.sp = got.dp, got.sp
    return fac


def _work(m):
    torch = _lib.require_cuda()
    return torch.empty(_lib.load().mt_work_doubles(ctypes.byref(m.desc)), dtype=torch.float64,
                       device=m.device)


def logdet(factor):
    """2 * sum log diag(L), FP64, fixed reduction order (factor.py:318-323)."""
    torch = _lib.require_cuda()
    m = factor.matrix
    out = torch.empty(1, dtype=torch.float64, device=m.device)
    _lib.check(_lib.load().mt_logdet(ctypes.byref(m.desc), _lib.ptr(_work(m)), _lib.ptr(out),
                                     _lib.stream_handle()), "mt_logdet")
    return float(out.item())


def _pad_rhs(factor, rhs):
    torch = _lib.require_cuda()
    x = np.array(rhs, dtype=np.float64, copy=True)
    vec = x.ndim == 1
    if vec:
        x = x[:, None]
    if x.ndim != 2 or x.shape[0] != factor.n:
        raise ValueError(f"rhs has {x.shape[0]} rows, factor has {factor.n}")
    npad = factor.p * factor.nb
    buf = np.zeros((npad, x.shape[1]))
    buf[: factor.n] = x
    return torch.from_numpy(buf).to(factor.matrix.device), vec, x.shape[1]


def solve(factor, rhs):
    """Solve (L L^T) x = rhs; rhs (n,) or (n, m) -> same shape (factor.py:292-315)."""
    d, vec, m = _pad_rhs(factor, rhs)
    _lib.check(_lib.load().mt_solve(ctypes.byref(factor.matrix.desc), _lib.ptr(d), m, 3,
                                    _lib.stream_handle()), "mt_solve")
    out = d.cpu().numpy()[: factor.n]
    return out[:, 0].copy() if vec else out


def forward_solve(factor, rhs):
    """y = L^{-1} rhs (the half-solve the likelihood's quadratic form needs)."""
    d, vec, m = _pad_rhs(factor, rhs)
    _lib.check(_lib.load().mt_solve(ctypes.byref(factor.matrix.desc), _lib.ptr(d), m, 1,
                                    _lib.stream_handle()), "mt_solve")
    out = d.cpu().numpy()[: factor.n]
    return out[:, 0].copy() if vec else out


def matvec_lower(factor, v):
    """L @ v (factor.py:326-340)."""
    v = np.asarray(v, dtype=np.float64)
    if v.shape != (factor.n,):
        raise ValueError(f"vector has shape {v.shape}, expected ({factor.n},)")
    d, _, _ = _pad_rhs(factor, v)
    out = d.clone()
    _lib.check(_lib.load().mt_matvec_lower(ctypes.byref(factor.matrix.desc), _lib.ptr(d),
                                           _lib.ptr(out), _lib.stream_handle()), "mt_matvec_lower")
    return out.cpu().numpy()[: factor.n, 0].copy()


def reconstruction_error(factor, reference):
    """||reference - L L^T||_F over the symmetric extent (factor.py:343-369).

    Diagnostic only: computed from the host views (not on the hot path).
    """
    n = factor.n
    low = np.zeros((n, n))
    for (i, j), t in factor.tiles.items():
        blk = t.dp
        low[factor.slice_of(i), factor.slice_of(j)] = np.tril(blk) if i == j else blk
    ref = reference.to_dense()
    r = ref - low @ low.T
    # absent (DST) tiles count as zero blocks of L, matching the reference
    return float(math.sqrt(float(np.sum(r * r))))


_ENGINES = {"ffma": 0, "tf32x3": 1, "tf32x3_rz": 2}


def set_fp32_engine(name):
    """Select the off-band (FP32) update engine (used when nb is a multiple of 256):

    * 'tf32x3' (default): tcgen05 3xTF32 with the TMEM accumulator restarted
      every 32 K-columns and the chunks summed in FP32 with round-to-nearest
      (FP32-accurate, like the reference's sgemm, factor.py:273-274);
    * 'tf32x3_rz': tcgen05 3xTF32 accumulating the whole K range in TMEM
      (the tensor core rounds each partial toward zero: a systematic bias;
      faster, opt-in);
    * 'ffma': SIMT FP32 FMA.
    Returns the previous engine name."""
    old = _lib.load().mt_set_option(0, _ENGINES[name])
    return {v: k for k, v in _ENGINES.items()}[old]


def set_legacy_dmma(flag):
    """1: use the register-staged DMMA band update instead of the TMA-staged one
    (A/B comparisons; both apply identical DMMA sequences). Returns the old flag."""
    return _lib.load().mt_set_option(2, int(flag))


def set_tc_trsm(flag):
    """1 (default): off-band panel TRSM as a tcgen05 3xTF32 GEMM against
    W = L_kk^{-1}; 0: SIMT blocked substitution. Returns the old flag."""
    return _lib.load().mt_set_option(3, int(flag))


def set_update_ctas(ctas):
    """Cap the CTAs of the bulk trailing update (0 = all SMs); returns the old cap."""
    return _lib.load().mt_set_option(1, int(ctas))
