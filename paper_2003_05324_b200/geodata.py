"""Synthetic inputs: datasets, seeded locations, Morton order, GPU field sampling.

Host-side input synthesis mirroring `mixtile.geodata` (geodata.py:19-249) so
that benchmarks and parity tests build bit-identical locations from the same
seeds without the reference installed.  `generate_field` samples Z = L v with
the full-DP factor computed on the GPU (the reference factors on the CPU,
geodata.py:88-106), which is what makes field-sampled z feasible at
N >= 65536.
"""

from dataclasses import dataclass, field

import numpy as np

from .covmath import DistanceMetric


@dataclass(frozen=True)
class GeoDataset:
    """n locations (n, 2) and one observation each (geodata.py:19-52)."""

    locations: np.ndarray
    z: np.ndarray
    metric: DistanceMetric = field(default_factory=DistanceMetric.euclidean)

    def __post_init__(self):
        locs = np.array(self.locations, dtype=np.float64)
        z = np.array(self.z, dtype=np.float64)
        if locs.ndim != 2 or locs.shape[1] != 2:
            raise ValueError(f"locations must be (n, 2), got {locs.shape}")
        if z.shape != (locs.shape[0],):
            raise ValueError("z length must match locations")
        if locs.shape[0] == 0:
            raise ValueError("dataset must contain at least one location")
        if not (np.isfinite(locs).all() and np.isfinite(z).all()):
            raise ValueError("dataset values must be finite")
        if self.metric.kind == "great_circle" and (np.abs(locs[:, 1]) > 90.0).any():
            raise ValueError("latitude outside [-90, 90]")
        locs.setflags(write=False)
        z.setflags(write=False)
        object.__setattr__(self, "locations", locs)
        object.__setattr__(self, "z", z)

    @property
    def n(self):
        return self.z.shape[0]

    def take(self, idx):
        idx = np.asarray(idx)
        return GeoDataset(self.locations[idx], self.z[idx], self.metric)


def derive_seed(seed, index):
    """Child seed from SeedSequence(seed, spawn_key=(index,)) (geodata.py:55-58)."""
    ss = np.random.SeedSequence(entropy=int(seed), spawn_key=(int(index),))
    return int(ss.generate_state(1, dtype=np.uint64)[0])


def _repeat_mask(locs):
    """True for every row equal to an earlier row in (x, y) lexicographic order."""
    order = np.lexsort((locs[:, 1], locs[:, 0]))
    s = locs[order]
    rep = np.zeros(len(locs), dtype=bool)
    rep[1:] = (s[1:] == s[:-1]).all(axis=1)
    out = np.zeros(len(locs), dtype=bool)
    out[order] = rep
    return out


def generate_locations(n, seed=0):
    """n distinct points uniform on the open unit square (geodata.py:61-74)."""
    if n < 1:
        raise ValueError(f"need n >= 1 locations, got {n}")
    rng = np.random.default_rng(seed)
    locs = rng.uniform(size=(n, 2))
    for _ in range(64):
        redraw = ((locs <= 0.0) | (locs >= 1.0)).any(axis=1) | _repeat_mask(locs)
        cnt = int(redraw.sum())
        if cnt == 0:
            return locs
        locs[redraw] = rng.uniform(size=(cnt, 2))
    raise RuntimeError("could not draw distinct interior locations")


def _interleave(v):
    v = v.astype(np.uint64)
    for shift, mask in ((16, 0x0000FFFF0000FFFF), (8, 0x00FF00FF00FF00FF),
                        (4, 0x0F0F0F0F0F0F0F0F), (2, 0x3333333333333333),
                        (1, 0x5555555555555555)):
        v = (v | (v << np.uint64(shift))) & np.uint64(mask)
    return v


def morton_keys(locations):
    """Z-order keys over the bounding box, 21 bits per axis (geodata.py:220-237)."""
    locs = np.asarray(locations, dtype=np.float64)
    q = []
    top = np.uint64(2 ** 21 - 1)
    for d in range(2):
        col = locs[:, d]
        lo, hi = float(col.min()), float(col.max())
        if hi - lo == 0.0:
            q.append(np.zeros(len(col), dtype=np.uint64))
        else:
            scaled = (col - lo) / (hi - lo) * float(2 ** 21 - 1)
            q.append(np.minimum(scaled.astype(np.uint64), top))
    return _interleave(q[0]) | (_interleave(q[1]) << np.uint64(1))


def morton_sort(dataset):
    """(dataset in Z order, permutation) with sorted.z == dataset.z[perm] (geodata.py:240-249)."""
    perm = np.argsort(morton_keys(dataset.locations), kind="stable")
    return dataset.take(perm), perm


def generate_field(locations, params, metric=None, seed=0, nb=256):
    """Z = L v, L the full-DP GPU Cholesky factor of the Matern covariance,
    v = default_rng(seed).standard_normal(n) (geodata.py:88-106)."""
    from . import factor as _factor
    from . import tilestore as _tilestore

    metric = metric or DistanceMetric.euclidean()
    locations = np.asarray(locations, dtype=np.float64)
    n = locations.shape[0]
    holder = GeoDataset(locations, np.zeros(n), metric)
    mat = _tilestore.assemble_covariance(holder, params, nb=min(nb, n),
                                         policy=_tilestore.PrecisionPolicy.dp())
    try:
        fac = _factor.cholesky(mat)
    except _factor.FactorizationError as exc:
        raise RuntimeError(f"covariance not positive definite: {exc}") from exc
    v = np.random.default_rng(seed).standard_normal(n)
    return GeoDataset(locations, _factor.matvec_lower(fac, v), metric)


@dataclass(frozen=True)
class FoldAssignment:
    """k-fold partition of n rows (geodata.py:114-121)."""

    k: int
    fold_of: np.ndarray
    folds: tuple

    @property
    def n(self):
        return self.fold_of.shape[0]


def kfold_split(n, k, seed=0):
    """Random partition into k folds whose sizes differ by at most one: the
    first n % k folds get one extra row; each fold's rows are sorted
    (geodata.py:124-146, same generator draws so folds match the reference)."""
    if n < 1:
        raise ValueError(f"need n >= 1, got {n}")
    if k < 2 or k > n:
        raise ValueError(f"need 2 <= k <= n, got k={k}, n={n}")
    perm = np.random.default_rng(seed).permutation(n)
    sizes = [n // k + (1 if f < n % k else 0) for f in range(k)]
    bounds = np.concatenate(([0], np.cumsum(sizes)))
    folds = tuple(np.sort(perm[bounds[f]:bounds[f + 1]]) for f in range(k))
    fold_of = np.empty(n, dtype=np.int64)
    for f, idx in enumerate(folds):
        fold_of[idx] = f
    return FoldAssignment(k=k, fold_of=fold_of, folds=folds)
