"""Quick phase timing of one likelihood evaluation (dev tool, not the bench)."""
import ctypes, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_05324_b200 as mt
from paper_2003_05324_b200 import _lib

def run(n, nb, pol, theta=(1.0, 0.1, 0.5), reps=2, lookahead=1):
    locs = mt.generate_locations(n, seed=1)
    ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.random.default_rng(2).standard_normal(n)))
    asm = mt.TileAssembler(ds, nb)
    ev = mt.Evaluator(asm, pol, lookahead=lookahead)
    m = ev.matrix
    lib = _lib.load(); st = _lib.stream_handle()
    th = _lib.matern_struct(*theta)
    for r in range(reps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        m.reset_status()
        e[0].record()
        _lib.check(lib.mt_generate(ctypes.byref(m.desc), _lib.ptr(asm.d_locs), 0, 0.0, ctypes.byref(th), st))
        e[1].record()
        _lib.check(lib.mt_cholesky(ctypes.byref(m.desc), lookahead, st))
        e[2].record()
        _lib.check(lib.mt_logdet(ctypes.byref(m.desc), _lib.ptr(ev.work), _lib.ptr(ev.out), st))
        _lib.check(lib.mt_quad(ctypes.byref(m.desc), _lib.ptr(asm.d_z), _lib.ptr(ev.work), _lib.ptr(ev.out[1:]), st))
        e[3].record()
        torch.cuda.synchronize()
        bad, ov, _ = m.read_status()
        tg, tc, ts = e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3])
        fl = n ** 3 / 3
        print(f"n={n} nb={nb} {pol.label()} la={lookahead}: gen {tg:.2f} ms chol {tc:.2f} ms ({fl/tc/1e9:.2f} TF/s) "
              f"logdet+quad {ts:.2f} ms  bad={bad} ov={ov} out={ev.out.tolist()}", flush=True)

if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    for pol in (mt.PrecisionPolicy.mp(diag_thick=2), mt.PrecisionPolicy.dp()):
        run(n, 512, pol)
    run(n, 512, mt.PrecisionPolicy.mp(diag_thick=2), lookahead=0, reps=1)
