"""A/B of library runtime options on the MP Cholesky (dev tool): for each
option setting, Cholesky ms (best of reps) at each N, plus (logdet, quad) to
confirm the variants agree bitwise.

usage: python tools/ab_opts.py OPT VAL1,VAL2,... [N1,N2,...] [t] [reps]
   e.g. python tools/ab_opts.py 6 0,4,8,16 65536,131072 8 3"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2003_05324_b200 as mt
from paper_2003_05324_b200 import _lib

opt = int(sys.argv[1])
vals = [int(v) for v in sys.argv[2].split(",")]
ns = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "65536").split(",")]
t = int(sys.argv[4]) if len(sys.argv) > 4 else 8
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
lib = _lib.load()
th = mt.MaternParams(1.0, 0.1, 0.5)
for n in ns:
    locs = mt.generate_locations(n, seed=mt.derive_seed(0, 0))
    ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.random.default_rng(1).standard_normal(n)))
    ev = mt.Evaluator(mt.TileAssembler(ds, 512), mt.PrecisionPolicy.mp(diag_thick=t))
    for rnd in range(2):  # two rounds: interleave to spread clock drift
        for v in vals:
            old = lib.mt_set_option(opt, v)
            ev(th)
            best, res = 1e30, None
            for _ in range(reps):
                e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                ev.launch(th, chol_events=e)
                res = ev.finish()
                best = min(best, e[0].elapsed_time(e[1]))
            lib.mt_set_option(opt, old)
            print(json.dumps({"n": n, "t": t, "opt": opt, "val": v, "round": rnd, "cholesky_ms": best,
                              "tflops": n ** 3 / 3 / best / 1e9, "logdet": res[0], "quad": res[1]}),
                  flush=True)
    del ev
    torch.cuda.empty_cache()
