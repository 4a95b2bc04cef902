"""CPU half of the configs[1]-scale parity golden (dev tool, build container):
the oracle port of the reference (bitwise-pinned on the small goldens)
evaluates DP, MP(t=2) and MP(t=8) log-likelihoods on the N=65536 field the
GPU drew (tools/make_field65536.py), timed like cli.py:247-258.  Writes
tests/golden/field65536.npz (z, results, the GPU's own values for the record);
the locations are regenerated from their seed by the test.

usage: python tools/golden65536_cpu.py gpurun_out/field65536_gpu.npz"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from threadpoolctl import threadpool_limits

from oracle import mixtile_oracle as O
import paper_2003_05324_b200.geodata as G

src = np.load(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/field65536_gpu.npz")
locs, z = src["locs"], src["z"]
n, nb = len(z), int(src["nb"])
th = tuple(float(v) for v in src["theta"])
# the locations are the seeded ones (tests/test_gpu_scale.py), Morton sorted
want_locs = G.morton_sort(G.GeoDataset(G.generate_locations(n, seed=G.derive_seed(2, 0)),
                                       np.zeros(n)))[0].locations
assert np.array_equal(locs, want_locs)
p = n // nb
res, secs = {}, {}
with threadpool_limits(limits=os.cpu_count()):
    for tag, mode, t in (("dp", "dp", p), ("mp:2", "mp", 2), ("mp:8", "mp", 8)):
        t0 = time.perf_counter()
        val, ld, q = O.loglik(locs, z, th, nb, mode, t)
        secs[tag] = time.perf_counter() - t0
        res[tag] = [val, ld, q]
        print(json.dumps({"tag": tag, "loglik": val, "logdet": ld, "quad": q,
                          "seconds": secs[tag]}), flush=True)
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "field65536.npz")
np.savez_compressed(out, z=z, theta=np.array(th), nb=np.array(nb),
                    results=np.array(json.dumps(res)),
                    gpu_results=src["gpu_results"],
                    meta=np.array(json.dumps({
                        "recipe": "locations generate_locations(65536, seed=derive_seed(2,0)); z = GPU "
                                  "full-DP generate_field(seed=derive_seed(2,1), nb=512); morton_sort",
                        "cpu": "oracle port (tools/golden65536_cpu.py), build container",
                        "cpu_seconds": secs, "cores": os.cpu_count()})))
print("wrote", out)
