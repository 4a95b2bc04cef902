"""GPU half of the configs[1]-scale parity golden (dev tool, run on a B200):
the field of tests/test_gpu_scale.py (N=65536, seed 2, Matern(1, 0.1, 0.5),
z = L v from the build's own full-DP generate_field), Morton
sorted, plus the GPU's DP / MP(t=2) / MP(t=8) log-likelihoods.  The CPU half
(tools/golden65536_cpu.py) evaluates the same inputs with the oracle port.

usage: python tools/make_field65536.py <out.npz>"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2003_05324_b200 as mt

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/field65536_gpu.npz"
th = mt.MaternParams(1.0, 0.1, 0.5)
locs = mt.generate_locations(65536, seed=mt.derive_seed(2, 0))
ds, _ = mt.morton_sort(mt.generate_field(locs, th, seed=mt.derive_seed(2, 1), nb=512))
res = {}
for tag, pol in (("dp", mt.PrecisionPolicy.dp()), ("mp:2", mt.PrecisionPolicy.mp(diag_thick=2)),
                 ("mp:8", mt.PrecisionPolicy.mp(diag_thick=8))):
    ev = mt.loglik(ds, th, 512, pol)
    res[tag] = [ev.value, ev.logdet, ev.quad]
    print(tag, res[tag], flush=True)
np.savez_compressed(out, locs=ds.locations, z=ds.z, theta=np.array(th.as_tuple()), nb=np.array(512),
                    gpu_results=np.array(json.dumps(res)))
