"""configs[4] CPU cross-check (dev tool, build container): the CPU reference
(oracle port) evaluates the profile log-likelihood at the GPU's DP MLE
theta-hat on the same N=65536 field (mle.py:102-114), as SURVEY.md 8d
prescribes (one CPU evaluation at the GPU theta-hat).

usage: python tools/mle_cpu_check.py gpurun_out/mle_config5_data.npz"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from threadpoolctl import threadpool_limits

from oracle import mixtile_oracle as O

d = np.load(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/mle_config5_data.npz")
fits = json.loads(str(d["fits"]))
locs, z, nb = d["locs"], d["z"], int(d["nb"])
n = len(z)
out = {"n": n, "nb": nb}
with threadpool_limits(limits=os.cpu_count()):
    for tag in ("dp",):
        th = fits[tag]["theta_hat"]
        t0 = time.perf_counter()
        val, ld, q, var = O.profile_loglik(locs, z, th[1], th[2], nb, "dp", n // nb)
        out[tag] = {"theta_hat": th, "gpu_profile_loglik": fits[tag]["loglik"],
                    "cpu_profile_loglik": val, "cpu_variance_opt": var,
                    "rel_diff": abs(val - fits[tag]["loglik"]) / abs(val),
                    "seconds": time.perf_counter() - t0}
        print(json.dumps(out[tag]), flush=True)
print(json.dumps(out))
