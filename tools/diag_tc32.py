"""Timing diagnostics of the bulk tcgen05 FP32 update (dev tool, WRONG results):
one step-0 trailing update over an MP matrix, epilogue variants via option 8."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_05324_b200 as mt
from paper_2003_05324_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
lib = _lib.load(); st = _lib.stream_handle()
ds = mt.GeoDataset(mt.generate_locations(n, seed=1), np.zeros(n))
asm = mt.TileAssembler(ds, 512)
m = mt.TileMatrix(n, 512, mt.PrecisionPolicy.mp(diag_thick=2))
asm.generate_into(m, mt.MaternParams(1.0, 0.1, 0.5))
m.split.normal_()  # any operands: timing only
d = ctypes.byref(m.desc)
p = m.p
tiles = sum(max(0, p - 2 - j) for j in range(2, p))
flops = tiles * 2.0 * 512 ** 3
for opts in os.environ.get("DIAG", "0,1,2,3,4,0").split(","):
    lib.mt_set_option(8, int(opts))
    for extra in (os.environ.get("EXTRA", "").split(";")):
        for kv in filter(None, extra.split(",")):
            k_, v_ = kv.split("=")
            lib.mt_set_option(int(k_), int(v_))
        ts = []
        for rep in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.check(lib.mt_update(d, 0, 2, p, st), "mt_update")
            e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = min(ts[1:])
        print(f"diag={opts} extra={extra!r}: {t:.3f} ms  {flops / t / 1e9:.1f} TF/s (3xTF32 FP32 products)", flush=True)
lib.mt_set_option(8, 0)
