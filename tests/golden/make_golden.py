"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Run in the build container only (the reference tree is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Each fixture stores inputs (locations, z, parameters) together with the
reference's own outputs, so the oracle restatement and the CUDA path can both
be checked against the reference without the reference being present.
The reference is imported read-only; nothing is copied from it.
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import mixtile  # noqa: E402
from mixtile import covmath, factor, geodata, mle, tilestore  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
PP = tilestore.PrecisionPolicy


def _policy(tag):
    if tag == "dp":
        return PP.dp()
    mode, t = tag.split(":")
    return PP.mp(diag_thick=int(t)) if mode == "mp" else PP.dst(diag_thick=int(t))


def _sim(n, seed, theta, nb=256, sort=True):
    locs = geodata.generate_locations(n, seed=geodata.derive_seed(seed, 0))
    ds = geodata.generate_field(locs, theta, seed=geodata.derive_seed(seed, 1), nb=nb)
    if sort:
        ds, _ = geodata.morton_sort(ds)
    return ds


def loglik_case(name, ds, theta, nb, tags):
    out = {"locs": ds.locations, "z": ds.z,
           "theta": np.array(theta.as_tuple()), "nb": np.array(nb)}
    meta = {}
    for tag in tags:
        pol = _policy(tag)
        try:
            ev = mle.loglik(ds, theta, nb, pol)
            meta[tag] = [ev.value, ev.logdet, ev.quad]
        except factor.FactorizationError as exc:
            meta[tag] = ["npd", exc.index]
    out["results"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(name, meta)


def factor_case(name, n, nb, tags, theta, seed):
    locs = geodata.generate_locations(n, seed=seed)
    z = np.random.default_rng(seed + 1).standard_normal(n)
    ds = geodata.GeoDataset(locs, z)
    out = {"locs": locs, "z": z, "theta": np.array(theta.as_tuple()), "nb": np.array(nb)}
    meta = {}
    for tag in tags:
        pol = _policy(tag)
        m = tilestore.assemble_covariance(ds, theta, nb, pol)
        asm_dense = m.to_dense()
        f = factor.cholesky(m)
        low = np.zeros((n, n))
        spmask = np.zeros((f.p, f.p), dtype=np.int8)
        for (i, j), t in f.tiles.items():
            blk = np.tril(t.dp) if i == j else t.dp
            low[f.slice_of(i), f.slice_of(j)] = blk
            spmask[i, j] = 1 if t.sp is not None else 0
        key = tag.replace(":", "")
        out[f"assembled_{key}"] = asm_dense
        out[f"lower_{key}"] = low
        out[f"spmask_{key}"] = spmask
        out[f"solve_{key}"] = factor.solve(f, z)
        meta[tag] = {"logdet": factor.logdet(f), "flops": [f.flops.dp, f.flops.sp]}
    out["results"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(name, {k: v["logdet"] for k, v in meta.items()})


def bessel_case():
    nus = np.array([0.05, 0.25, 0.5, 0.8, 1.0, 1.5, 1.7, 2.5, 3.3, 5.0])
    xs = np.concatenate([10.0 ** np.linspace(-6, 0.3, 40), np.linspace(2.0, 2.0, 1),
                         np.linspace(2.0001, 60.0, 60)])
    vals = np.stack([covmath.bessel_k_array(float(nu), xs) for nu in nus])
    r = np.concatenate([[0.0], 10.0 ** np.linspace(-5, 0.5, 80)])
    mat = {}
    for nu in (0.3, 0.5, 1.0, 1.5, 2.8):
        mat[str(nu)] = covmath.matern_array(r, covmath.MaternParams(1.7, 0.13, nu))
    gam_x = np.linspace(0.02, 12.0, 200)
    gam = np.array([covmath.gamma(float(x)) for x in gam_x])
    np.savez_compressed(os.path.join(OUT, "bessel.npz"), nus=nus, xs=xs, vals=vals, r=r,
                        gam_x=gam_x, gam=gam,
                        **{f"matern_{k}": v for k, v in mat.items()})
    print("bessel", vals.shape)


def assembly_case():
    """Assembled tiles (dense, FP64 view) under several policies, both metrics."""
    out = {}
    rng = np.random.default_rng(5)
    for metric_name, metric in (("euc", covmath.DistanceMetric.euclidean()),
                                ("gc", covmath.DistanceMetric.great_circle())):
        if metric_name == "euc":
            locs = geodata.generate_locations(45, seed=11)
        else:
            locs = np.column_stack([rng.uniform(-20, 20, 45), rng.uniform(-60, 60, 45)])
        ds = geodata.GeoDataset(locs, np.zeros(45), metric)
        rng_ = 0.2 if metric_name == "euc" else 900.0
        for nu in (0.5, 1.0, 1.5, 0.35):
            th = covmath.MaternParams(1.3, rng_, nu)
            for tag in ("dp", "mp:2", "dst:2"):
                m = tilestore.assemble_covariance(ds, th, 8, _policy(tag))
                out[f"{metric_name}_{nu}_{tag.replace(':', '')}"] = m.to_dense()
        out[f"{metric_name}_locs"] = locs
    np.savez_compressed(os.path.join(OUT, "assembly.npz"), **out)
    print("assembly", len(out))


def flops_case():
    rows = []
    for n, nb, tag in [(64, 8, "dp"), (64, 8, "mp:2"), (128, 8, "mp:2"), (1024, 64, "mp:2"),
                       (37, 8, "mp:1"), (4096, 256, "mp:2"), (65536, 512, "mp:2"),
                       (64, 8, "dst:1"), (100, 7, "dst:3")]:
        fl = factor.planned_flops(n, nb, _policy(tag))
        rows.append([n, nb, tag, fl.dp, fl.sp])
    with open(os.path.join(OUT, "flops.json"), "w") as fh:
        json.dump(rows, fh, indent=1)
    print("flops", rows)


def fit_case():
    theta = covmath.MaternParams(1.0, 0.1, 0.5)
    ds = _sim(200, 3, theta, nb=64)
    out = {"locs": ds.locations, "z": ds.z}
    meta = {}
    for tag in ("dp", "mp:1"):
        res = mle.fit_matern(ds, 32, _policy(tag))
        meta[tag] = {"params": list(res.params.as_tuple()), "value": res.value,
                     "evaluations": res.evaluations, "iterations": res.iterations,
                     "trace": [[tp.spatial_range, tp.smoothness, tp.value] for tp in res.trace]}
    out["results"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(OUT, "fit_small.npz"), **out)
    print("fit", {k: v["params"] for k, v in meta.items()})


def krige_case():
    """predict.krige / pmse_kfold outputs of the reference (predict.py:37-92)."""
    from mixtile import predict
    out = {}
    meta = {}
    th = covmath.MaternParams(1.4, 0.12, 1.5)
    ds = _sim(300, 5, th, nb=64, sort=False)
    test = geodata.generate_locations(37, seed=99)
    out.update(locs=ds.locations, z=ds.z, test=test, theta=np.array(th.as_tuple()))
    for tag in ("dp", "mp:1", "mp:2"):
        out[f"pred_{tag.replace(':', '_')}"] = predict.krige(ds, test, th, 64, _policy(tag))
    th2 = covmath.MaternParams(1.0, 0.1, 0.5)
    ds2 = _sim(200, 6, th2, nb=64, sort=False)
    out.update(locs2=ds2.locations, z2=ds2.z)
    rep = predict.pmse_kfold(ds2, th2, 32, _policy("mp:1"), k=5, seed=3)
    out["pmse_pred"] = rep.predictions
    meta["pmse"] = rep.pmse
    meta["fold_mse"] = list(rep.fold_mse)
    folds = geodata.kfold_split(23, 4, seed=7)
    out["fold_of_23_4_7"] = folds.fold_of
    out["results"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(OUT, "krige.npz"), **out)
    print("krige", meta)


def strong_npd_case():
    """configs[2]-shaped field at N=16384: the reference's MP (t=8) is indefinite;
    record its FactorizationError index (the GPU RN engine must match it)."""
    n = 16384
    locs = geodata.generate_locations(n, seed=geodata.derive_seed(3, 0))
    ds, _ = geodata.morton_sort(geodata.GeoDataset(locs, np.random.default_rng(3).standard_normal(n)))
    try:
        mle.loglik(ds, covmath.MaternParams(1.0, 0.3, 1.0), 512, PP.mp(diag_thick=8))
        idx = None
    except factor.FactorizationError as exc:
        idx = exc.index
    json.dump({"recipe": "generate_locations(16384, seed=derive_seed(3,0)); z = default_rng(3)."
                         "standard_normal(n); morton_sort; loglik(theta=(1.0, 0.3, 1.0), nb=512, "
                         "PrecisionPolicy.mp(diag_thick=8))",
               "n": n, "nb": 512, "theta": [1.0, 0.3, 1.0], "band_t": 8,
               "reference_factorization_error_index": idx},
              open(os.path.join(OUT, "strong16384_npd.json"), "w"), indent=1)
    print("strong16384 npd", idx)


def main():
    print("reference mixtile", mixtile.__version__)
    th1 = covmath.MaternParams(1.0, 0.1, 0.5)
    # config 1 of BASELINE.json: N=4096, nb=256, theta=(1, 0.1, 0.5), seed s=0
    ds1 = _sim(4096, 0, th1, nb=256)
    loglik_case("config1", ds1, th1, 256, ["dp", "mp:1", "mp:2", "mp:4", "mp:8", "mp:16"])
    # strong-correlation field, general nu (config-3 shape, small N)
    th3 = covmath.MaternParams(1.0, 0.3, 1.0)
    ds3 = _sim(1024, 3, th3, nb=128)
    loglik_case("strong1024", ds3, th3, 128, ["dp", "mp:1", "mp:2", "mp:4"])
    # ragged tiling and a general-nu field
    th4 = covmath.MaternParams(1.5, 0.12, 0.8)
    ds4 = _sim(1000, 4, th4, nb=96)
    loglik_case("ragged1000", ds4, th4, 96, ["dp", "mp:1", "mp:3", "dst:3"])
    factor_case("factor_small", 70, 8, ["dp", "mp:1", "mp:2", "mp:9", "dst:2"], th1, 7)
    bessel_case()
    assembly_case()
    flops_case()
    fit_case()
    krige_case()
    strong_npd_case()


if __name__ == "__main__":
    main()
