"""One band-update step: TMA DMMA vs register-staged, per sub-tile diff (dev tool)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_05324_b200 as mt
from paper_2003_05324_b200 import _lib

lib = _lib.load(); st = _lib.stream_handle()
for variant in (0,):
  for n, nb, t, k in [(4096, 256, 8, 0), (4096, 256, 8, 3), (8192, 512, 2, 0), (8192, 512, 8, 1), (16384, 512, 8, 0), (16384, 512, 8, 2)]:
      locs = mt.generate_locations(n, seed=5)
      ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.zeros(n)))
      pol = mt.PrecisionPolicy.mp(diag_thick=t)
      m = mt.assemble_covariance(ds, mt.MaternParams(1.0, 0.1, 0.5), nb, pol)
      d = ctypes.byref(m.desc)
      mt.set_legacy_dmma(1)
      for kk in range(k):
          lib.mt_panel(d, kk, st); lib.mt_update(d, kk, kk + 1, m.p, st)
      lib.mt_panel(d, k, st)
      torch.cuda.synchronize()
      dp0, sp0 = m.dp_pool.clone(), m.sp_pool.clone()
      res = []
      for legacy in (1, variant):
          m.dp_pool.copy_(dp0); m.sp_pool.copy_(sp0)
          mt.set_legacy_dmma(legacy)
          _lib.check(lib.mt_update(d, k, k + 1, m.p, st), "upd")
          torch.cuda.synchronize()
          res.append(m.dp_pool.clone().cpu().numpy())
      mt.set_legacy_dmma(0)
      te = nb * nb
      p = m.p
      bad = []
      slot = 0
      for j in range(p):
          for i in range(j, min(p, j + t)):
              a = res[0][slot * te:(slot + 1) * te].reshape(nb, nb)
              b = res[1][slot * te:(slot + 1) * te].reshape(nb, nb)
              if not np.array_equal(a, b):
                  dd = np.abs(a - b)
                  subs = sorted({(r // 128, c // 64) for r, c in zip(*np.nonzero(dd))})
                  kinds = ("F64" if i - k < t else "F32", "F64" if j - k < t else "F32")
                  bad.append(((i, j), kinds, float(dd.max()), subs[:6], len(subs)))
              slot += 1
      print("variant", variant, n, nb, t, "k=", k, "bad tiles", len(bad), flush=True)
      for b in bad[:12]:
          print("   ", b)
