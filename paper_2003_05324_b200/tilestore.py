"""Device-resident tile grid, precision policy and covariance assembly.

Mirrors `mixtile.tilestore` (tilestore.py:20-262).  The payloads live in HBM
in two pools (FP64 band, FP32 off-band; see include/mixtile_b200.h for the
layout); `TileMatrix.tiles` is a lazy host *view* with the reference's
`Tile(dp, sp)` objects (Fortran-ordered numpy arrays) materialised on access,
for tests and inspection only -- the compute path never touches it.
"""

import ctypes
import math
import warnings
import weakref
from collections.abc import Mapping
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _lib


class PrecisionOverflowError(ValueError):
    """An FP64 value exceeded FP32 range while narrowing (tilestore.py:20-21)."""


class Mode(Enum):
    DP = "dp"
    MP = "mp"
    DST = "dst"


def percent_to_thickness(dp_percent, p):
    """t = max(1, floor(p * pct / 100 + 1/2)) for pct in (0, 100] (tilestore.py:33-43)."""
    if not (0.0 < dp_percent <= 100.0):
        raise ValueError(f"dp_percent must be in (0, 100], got {dp_percent}")
    if p < 1:
        raise ValueError(f"need p >= 1, got {p}")
    return max(1, int(math.floor(p * dp_percent / 100.0 + 0.5)))


@dataclass(frozen=True)
class PrecisionPolicy:
    """Mode plus band thickness, resolved against a tile order p (tilestore.py:46-89)."""

    mode: Mode
    diag_thick: int = None
    dp_percent: float = None

    @classmethod
    def dp(cls):
        return cls(Mode.DP)

    @classmethod
    def mp(cls, diag_thick=None, dp_percent=None):
        return cls(Mode.MP, diag_thick, dp_percent)

    @classmethod
    def dst(cls, diag_thick=None, dp_percent=None):
        return cls(Mode.DST, diag_thick, dp_percent)

    def resolve(self, p):
        if self.mode is Mode.DP:
            return PrecisionPolicy(Mode.DP, p, self.dp_percent)
        if self.diag_thick is not None:
            t = int(self.diag_thick)
            if not (1 <= t <= p):
                raise ValueError(f"diag_thick must be in [1, {p}], got {t}")
            return PrecisionPolicy(self.mode, t, self.dp_percent)
        if self.dp_percent is not None:
            return PrecisionPolicy(self.mode, percent_to_thickness(self.dp_percent, p),
                                   self.dp_percent)
        raise ValueError("policy needs diag_thick or dp_percent to resolve")

    def label(self):
        if self.mode is Mode.DP:
            return "dp"
        tag = f"{self.dp_percent:g}" if self.dp_percent is not None else f"t{self.diag_thick}"
        return f"{self.mode.value}:{tag}"


def band_member(i, j, policy):
    """Tile (i, j) is FP64 iff |i - j| < diag_thick (tilestore.py:92-96)."""
    if policy.mode.value == "dp":
        return True
    return abs(i - j) < policy.diag_thick


class Tile:
    """Host view of one tile: FP64 payload, FP32 payload, or both."""

    __slots__ = ("dp", "sp")

    def __init__(self, dp=None, sp=None):
        self.dp = dp
        self.sp = sp


class _TileView(Mapping):
    """Lazy {(i, j): Tile} view over the device pools (reference: the tiles dict)."""

    def __init__(self, owner):
        # weak: the matrix owns the view; a strong back-reference would form a
        # cycle that keeps the (possibly 100+ GB) device pools alive after `del`
        self._m = weakref.proxy(owner)
        self._cache = {}

    def _keys(self):
        m = self._m
        for j in range(m.col_offset, m.p, m.col_stride):  # owned tile columns
            for i in range(j, m.p):
                if (i - m.row_offset) % m.row_stride == 0 and (
                        m.policy.mode.value != "dst" or i - j < m.policy.diag_thick):
                    yield (i, j)

    def __iter__(self):
        return self._keys()

    def __len__(self):
        return sum(1 for _ in self._keys())

    def __contains__(self, key):
        try:
            i, j = key
        except (TypeError, ValueError):
            return False
        m = self._m
        return (0 <= j <= i < m.p and (j - m.col_offset) % m.col_stride == 0
                and j >= m.col_offset and i >= m.row_offset
                and (i - m.row_offset) % m.row_stride == 0
                and (m.policy.mode.value != "dst" or i - j < m.policy.diag_thick))

    def __getitem__(self, key):
        if key not in self:
            raise KeyError(key)
        if self._m._version != self._cache.get("_v"):
            self._cache = {"_v": self._m._version}
        if key not in self._cache:
            self._cache[key] = self._m._host_tile(*key)
        return self._cache[key]


class TileMatrix:
    """Lower tile grid of an n x n symmetric matrix, resident on the GPU.

    Constructor arguments follow tilestore.TileMatrix(n, nb, policy); the
    reference's optional `tiles` dict is replaced by device pools allocated
    here (use `from_dense` to upload explicit payloads).
    """

    def __init__(self, n, nb, policy, device=None, col_stride=1, col_offset=0, row_stride=1,
                 row_offset=0, panel_slots=2):
        if n < 1:
            raise ValueError(f"need n >= 1, got {n}")
        if nb < 1:
            raise ValueError(f"need nb >= 1, got {nb}")
        torch = _lib.require_cuda()
        self.n = int(n)
        self.nb = int(nb)
        self.p = -(-self.n // self.nb)
        self.policy = policy.resolve(self.p)
        self.duplicate_locations = False
        self.factored = False
        self._version = 0
        # multi-GPU, P x Q block-cyclic: this rank stores the tiles (i, j) with
        # j = col_offset (mod col_stride = Q) and i = row_offset (mod row_stride = P)
        self.col_stride, self.col_offset = int(col_stride), int(col_offset)
        self.row_stride, self.row_offset = int(row_stride), int(row_offset)
        multi = self.col_stride > 1 or self.row_stride > 1
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        lib = _lib.load()
        mode = _lib.MODE_CODE[self.policy.mode.value]
        t = self.policy.diag_thick
        te = self.nb * self.nb
        ndp, nsp = ctypes.c_int64(), ctypes.c_int64()
        lib.mt_local_tiles_ex(self.p, t, mode, self.row_stride, self.row_offset, self.col_stride,
                              self.col_offset, ctypes.byref(ndp), ctypes.byref(nsp))
        ndp, nsp = ndp.value, nsp.value
        # rings of panels in flight: 2 slots (lookahead 1) or 3 (lookahead 2)
        self.panel_slots = max(2, int(panel_slots))
        nsc, nsl, ndpn = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        lib.mt_ring_tiles(self.p, t, mode, self.nb, self.row_stride, self.col_stride,
                          self.panel_slots, ctypes.byref(nsc), ctypes.byref(nsl), ctypes.byref(ndpn))
        nsc, ndpn = nsc.value, ndpn.value
        nsl = nsl.value if self.nb % 256 == 0 else 0
        self.dp_pool = torch.empty(max(ndp, 1) * te, dtype=torch.float64, device=dev)
        self.sp_pool = torch.empty(max(nsp, 1) * te, dtype=torch.float32, device=dev)
        self.scratch = torch.empty(max(nsc, 1) * te, dtype=torch.float32, device=dev)
        self.split = (torch.empty(nsl * te, dtype=torch.float32, device=dev) if nsl else None)
        self.dpanel = None
        if multi:
            self.dpanel = torch.empty(ndpn * te, dtype=torch.float64, device=dev)
        self.status = torch.empty(4, dtype=torch.int64, device=dev)
        self.desc = _lib.MtTiles(self.n, self.nb, self.p, t, mode, self.dp_pool.data_ptr(),
                                 self.sp_pool.data_ptr(), self.scratch.data_ptr(),
                                 self.status.data_ptr(),
                                 self.split.data_ptr() if self.split is not None else 0,
                                 self.col_stride, self.col_offset,
                                 self.dpanel.data_ptr() if self.dpanel is not None else 0,
                                 self.row_stride, self.row_offset, self.panel_slots)
        self.reset_status()
        self.tiles = _TileView(self)

    # -- geometry (tilestore.py:157-165) --------------------------------------
    def rows_of(self, i):
        return min(self.nb, self.n - i * self.nb)

    def slice_of(self, i):
        return slice(i * self.nb, i * self.nb + self.rows_of(i))

    def band(self, i, j):
        return band_member(i, j, self.policy)

    def tile(self, i, j):
        return self.tiles.get((i, j))

    @property
    def device(self):
        return self.dp_pool.device

    # -- device status -------------------------------------------------------
    def reset_status(self):
        _lib.check(_lib.load().mt_reset_status(ctypes.byref(self.desc), _lib.stream_handle()),
                   "mt_reset_status")

    def read_status(self):
        """(bad_pivot, overflow_count, duplicate_pairs); synchronises the stream."""
        bp, ov, du = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        rc = _lib.load().mt_read_status(ctypes.byref(self.desc), ctypes.byref(bp),
                                        ctypes.byref(ov), ctypes.byref(du), _lib.stream_handle())
        if rc not in (_lib.MT_OK, _lib.MT_E_NOT_SPD, _lib.MT_E_OVERFLOW):
            _lib.check(rc, "mt_read_status")
        return bp.value, ov.value, du.value

    # -- host view -------------------------------------------------------------
    def _download(self, i, j, which):
        shape = (self.rows_of(i), self.rows_of(j))
        out = np.empty(shape, dtype=np.float64 if which == 0 else np.float32, order="F")
        _lib.check(_lib.load().mt_get_tile(ctypes.byref(self.desc), i, j, which, _lib.np_ptr(out),
                                           _lib.stream_handle()), "mt_get_tile")
        return out

    def _host_tile(self, i, j):
        band = self.band(i, j)
        if band:
            dp = self._download(i, j, 0)
            sp = None
            t, p = self.policy.diag_thick, self.p
            # narrowed mirror of a band panel tile that fed FP32 updates
            # (factor.py:261-262): the device mirror is exactly RN(dp)
            if (self.factored and self.policy.mode.value == "mp" and i != j and i + t <= p - 1):
                sp = np.asfortranarray(dp, dtype=np.float32)
            return Tile(dp=dp, sp=sp)
        sp = self._download(i, j, 1)
        dp = np.asfortranarray(sp, dtype=np.float64) if self.factored else None
        return Tile(dp=dp, sp=sp)

    def _touch(self):
        self._version += 1

    def to_dense(self):
        """Full symmetric FP64 reconstruction; absent tiles read as zero (tilestore.py:167-179)."""
        out = np.zeros((self.n, self.n))
        for (i, j), t in self.tiles.items():
            blk = t.dp if t.dp is not None else t.sp.astype(np.float64)
            si, sj = self.slice_of(i), self.slice_of(j)
            if i == j:
                out[si, sj] = np.tril(blk) + np.tril(blk, -1).T
            else:
                out[si, sj] = blk
                out[sj, si] = blk.T
        return out

    def dump_csv(self, path):
        with open(path, "w", newline="") as fh:
            for row in self.to_dense():
                fh.write(",".join(repr(float(v)) for v in row) + "\n")

    @classmethod
    def from_dense(cls, a, nb, policy):
        """Tile a dense symmetric matrix (lower triangle read) and upload (tilestore.py:188-205)."""
        a = np.asarray(a, dtype=np.float64)
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise ValueError(f"need a square matrix, got {a.shape}")
        m = cls(a.shape[0], nb, policy)
        lib = _lib.load()
        st = _lib.stream_handle()
        for i in range(m.p):
            si = m.slice_of(i)
            for j in range(i + 1):
                blk = a[si, m.slice_of(j)]
                if m.band(i, j):
                    buf = np.asfortranarray(blk)
                    which = 0
                elif m.policy.mode.value == "mp":
                    with np.errstate(over="ignore"):
                        buf = np.asfortranarray(blk, dtype=np.float32)
                    if (np.isfinite(blk) & ~np.isfinite(buf)).any():
                        raise PrecisionOverflowError(
                            "value(s) exceed FP32 range during narrowing")
                    which = 1
                else:
                    continue
                _lib.check(lib.mt_put_tile(ctypes.byref(m.desc), i, j, which, _lib.np_ptr(buf), st),
                           "mt_put_tile")
        m._touch()
        return m


class TileAssembler:
    """Covariance assembly for one dataset and tile size (tilestore.py:212-253).

    Locations are uploaded once and stay resident across parameter values
    (the reference caches an O(N^2) distance dict instead); the duplicate
    scan runs once here, as the reference's distance pass does.
    """

    def __init__(self, dataset, nb):
        torch = _lib.require_cuda()
        self.dataset = dataset
        self.nb = int(nb)
        self.n = dataset.n
        self.p = -(-self.n // self.nb)
        dev = torch.device("cuda", torch.cuda.current_device())
        npad = self.p * self.nb
        # pinned staging (torch's caching host allocator) -> async H2D
        stage = torch.zeros((npad, 3), dtype=torch.float64, pin_memory=True)
        sv = stage.numpy()
        sv[: self.n, :2] = dataset.locations
        sv[: self.n, 2] = dataset.z
        d = stage.to(dev, non_blocking=True)
        self.d_locs = d[:, :2].contiguous()
        self.d_z = d[:, 2].contiguous()
        self.metric_code = _lib.METRIC_CODE[dataset.metric.kind]  # duck-typed: reference metrics too
        self.radius = float(dataset.metric.radius)
        probe = _Probe(self.n, self.nb, dev)
        _lib.check(_lib.load().mt_scan_duplicates(ctypes.byref(probe.desc), _lib.ptr(self.d_locs),
                                                  self.metric_code, self.radius,
                                                  _lib.stream_handle()), "mt_scan_duplicates")
        self.duplicate_locations = probe.read_dups() > 0
        if self.duplicate_locations:
            warnings.warn("dataset contains duplicate locations; the covariance "
                          "is singular", RuntimeWarning, stacklevel=2)

    def generate_into(self, m, params):
        th = _lib.matern_struct(*params.as_tuple())
        _lib.check(_lib.load().mt_generate(ctypes.byref(m.desc), _lib.ptr(self.d_locs),
                                           self.metric_code, self.radius, ctypes.byref(th),
                                           _lib.stream_handle()), "mt_generate")
        m._touch()

    def assemble(self, params, policy):
        m = TileMatrix(self.n, self.nb, policy)
        m.duplicate_locations = self.duplicate_locations
        self.generate_into(m, params)
        _, overflow, _ = m.read_status()
        if overflow:
            raise PrecisionOverflowError(
                f"{overflow} value(s) exceed FP32 range during narrowing")
        return m


class _Probe:
    """Minimal 1-tile descriptor carrying a status word for layout-free kernels."""

    def __init__(self, n, nb, dev):
        import torch
        self.status = torch.tensor([-1, 0, 0, 0], dtype=torch.int64, device=dev)
        self.dummy = torch.empty(1, dtype=torch.float64, device=dev)
        p = -(-n // nb)
        self.desc = _lib.MtTiles(n, nb, p, p, 0, self.dummy.data_ptr(), 0,
                                 self.dummy.data_ptr(), self.status.data_ptr(), 0)

    def read_dups(self):
        return int(self.status[2].item())


def assemble_covariance(dataset, params, nb, policy):
    """One-shot assembly (tilestore.py:256-262)."""
    return TileAssembler(dataset, nb).assemble(params, policy)
