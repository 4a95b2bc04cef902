"""Matern parameters, distance metrics and device Matern evaluation.

Mirrors the reference `mixtile.covmath` interface (covmath.py:33-358) for the
pieces the hot path needs.  Parameter/metric types are plain host data;
Matern values are computed on the GPU by the same device function the tile
generator uses (csrc/gen.cu), so `matern_array` here is a probe of exactly
the code that fills the covariance tiles.
"""

import math
from dataclasses import dataclass

import numpy as np

from . import _lib

EARTH_RADIUS_KM = 6371.0


@dataclass(frozen=True)
class MaternParams:
    """(variance, spatial_range, smoothness), each finite and > 0 (covmath.py:228-258)."""

    variance: float
    spatial_range: float
    smoothness: float

    def __post_init__(self):
        for name in ("variance", "spatial_range", "smoothness"):
            v = getattr(self, name)
            ok = isinstance(v, (int, float, np.floating, np.integer)) and math.isfinite(v) and v > 0
            if not ok:
                raise ValueError(f"MaternParams.{name} must be finite and > 0, got {v}")
            object.__setattr__(self, name, float(v))

    def as_tuple(self):
        return (self.variance, self.spatial_range, self.smoothness)

    def to_text(self):
        return ",".join(repr(v) for v in self.as_tuple())

    @classmethod
    def from_text(cls, text):
        parts = [s.strip() for s in text.split(",")]
        if len(parts) != 3:
            raise ValueError(f"expected 'variance,range,smoothness', got {text!r}")
        try:
            return cls(*(float(s) for s in parts))
        except ValueError as exc:
            raise ValueError(f"bad Matern parameter in {text!r}") from exc


@dataclass(frozen=True)
class DistanceMetric:
    """Euclidean plane or great circle of a radius; (lon, lat) degrees (covmath.py:299-317)."""

    kind: str
    radius: float = 0.0

    @classmethod
    def euclidean(cls):
        return cls("euclidean")

    @classmethod
    def great_circle(cls, radius=EARTH_RADIUS_KM):
        if not (radius > 0.0 and math.isfinite(radius)):
            raise ValueError(f"great-circle radius must be > 0, got {radius}")
        return cls("great_circle", float(radius))

    @property
    def code(self):
        return _lib.METRIC_CODE[self.kind]


def matern_array(r, params, use_closed_forms=True):
    """Matern covariance at distances r, evaluated on the GPU (covmath.py:261-283).

    use_closed_forms=False forces the general Bessel route even at nu = 1/2
    and 3/2 (the reference's switch for exercising the Bessel machinery)."""
    torch = _lib.require_cuda()
    r = np.asarray(r, dtype=np.float64)
    if r.size and np.min(r) < 0.0:
        raise ValueError("matern requires r >= 0")
    flat = np.ascontiguousarray(r.reshape(-1))
    d_r = torch.from_numpy(flat).cuda()
    d_out = torch.empty_like(d_r)
    th = _lib.matern_struct(*params.as_tuple())
    if not use_closed_forms:
        th.kind = 2  # Bessel route; its constants are prepared for every nu
    _lib.check(_lib.load().mt_matern_array(_lib.ptr(d_r), flat.size, th, _lib.ptr(d_out),
                                           _lib.stream_handle()), "mt_matern_array")
    return d_out.cpu().numpy().reshape(r.shape)


def matern(r, params):
    """Scalar Matern covariance, C(0) = variance exactly."""
    if not (r >= 0.0):
        raise ValueError(f"matern requires r >= 0, got {r}")
    if r == 0.0:
        return params.variance
    return float(matern_array(np.array([r]), params)[0])
