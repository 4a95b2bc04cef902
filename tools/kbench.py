"""Serialized per-kernel profile of one Cholesky (lookahead 0: no stream overlap,
so the event times are pure kernel durations)."""
import argparse, ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_05324_b200 as mt
from paper_2003_05324_b200 import _lib

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=65536); ap.add_argument("--nb", type=int, default=512)
ap.add_argument("--t", type=int, default=2); ap.add_argument("--dp", action="store_true")
ap.add_argument("--lookahead", type=int, default=0); ap.add_argument("--engine", default="tf32x3")
ap.add_argument("--legacy-dmma", type=int, default=0); ap.add_argument("--tc-trsm", type=int, default=1)
ap.add_argument("--pcol", type=int, default=-1); ap.add_argument("--yield-sms", type=int, default=-1)
ap.add_argument("--super", type=int, default=-1, help="option 6: super-column width (0 = slot order)")
a = ap.parse_args()
ap2 = None
if a.super >= 0:
    _lib.load().mt_set_option(6, a.super)
import os as _os
if _os.environ.get("MT_OPTS"):  # e.g. MT_OPTS=7=0,5=16
    for kv in _os.environ["MT_OPTS"].split(","):
        k_, v_ = kv.split("=")
        _lib.load().mt_set_option(int(k_), int(v_))
mt.set_fp32_engine(a.engine)
mt.set_legacy_dmma(a.legacy_dmma)
mt.set_tc_trsm(a.tc_trsm)
if a.pcol >= 0:
    _lib.load().mt_set_option(4, a.pcol)
if a.yield_sms >= 0:
    _lib.load().mt_set_option(5, a.yield_sms)
KINDS = ["gen64", "gen32", "potrf", "trsm64", "trsm32", "upd64", "upd32", "solve", "misc", "upd64p", "upd32p"]
locs = mt.generate_locations(a.n, seed=1)
ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.zeros(a.n)))
pol = mt.PrecisionPolicy.dp() if a.dp else mt.PrecisionPolicy.mp(diag_thick=a.t)
asm = mt.TileAssembler(ds, a.nb)
m = mt.TileMatrix(a.n, a.nb, pol)
lib = _lib.load(); st = _lib.stream_handle()
th = _lib.matern_struct(1.0, 0.1, 0.5)
for rep in range(2):
    m.reset_status()
    lib.mt_generate(ctypes.byref(m.desc), _lib.ptr(asm.d_locs), 0, 0.0, ctypes.byref(th), st)
    torch.cuda.synchronize()
    lib.mt_prof_begin(20000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lib.mt_cholesky(ctypes.byref(m.desc), a.lookahead, st)
    e1.record(); torch.cuda.synchronize()
    K = len(KINDS); arr = [(ctypes.c_double * K)() for _ in range(3)]; cnt = (ctypes.c_int64 * K)()
    lib.mt_prof_end(K, arr[0], arr[1], arr[2], cnt)
tot = e0.elapsed_time(e1)
print(f"n={a.n} nb={a.nb} {pol.label()} la={a.lookahead} super={a.super} opts={_os.environ.get('MT_OPTS', '')} legacy_dmma={a.legacy_dmma} tc_trsm={a.tc_trsm} pcol={a.pcol} yield={a.yield_sms} cholesky {tot:.1f} ms = {a.n**3/3/tot/1e9:.1f} TF/s  status={m.read_status()}")
for q in range(K):
    if cnt[q]:
        print(f"  {KINDS[q]:7s} launches={cnt[q]:5d} total={arr[0][q]:9.2f} ms avg={arr[0][q]/cnt[q]*1e3:9.1f} us  "
              f"{arr[1][q]/max(arr[0][q],1e-9)/1e9:8.2f} TF/s  {arr[2][q]/max(arr[0][q],1e-9)/1e6:8.1f} GB/s")
