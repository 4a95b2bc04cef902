"""CPU: host logic of the multi-GPU path (no GPU needed).

1. The rank-local pool layout of libmixtile_b200 (closed-form column starts,
   mt_local_tiles) against brute-force counting.
2. The distributed protocol -- `distributed.schedule`, column ownership and
   the panel broadcast -- executed by world_size-2 gloo processes with a
   test-only numpy tile backend (the oracle's LAPACK/BLAS calls).  The
   distributed factor, logdet and quad must equal the single-process oracle
   bit for bit, which is what the GPU ranks guarantee for their kernels too.
"""

import ctypes
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp
from scipy.linalg import blas as B
from scipy.linalg import lapack as LP

from oracle import mixtile_oracle as O
from paper_2003_05324_b200 import _lib
from paper_2003_05324_b200.distributed import owner, schedule


@pytest.mark.parametrize("p,t,mode", [(16, 2, 1), (16, 16, 0), (9, 3, 1), (7, 1, 1), (12, 4, 2),
                                      (1, 1, 0)])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_local_layout_matches_bruteforce(p, t, mode, world):
    lib = _lib.load()
    tot_dp = tot_sp = 0
    for r in range(world):
        ndp, nsp = ctypes.c_int64(), ctypes.c_int64()
        lib.mt_local_tiles(p, t, mode, world, r, ctypes.byref(ndp), ctypes.byref(nsp))
        cols = range(r, p, world)
        want_dp = sum(min(t if mode else p, p - j) for j in cols)
        want_sp = sum(max(0, p - t - j) for j in cols) if mode == 1 else 0
        assert (ndp.value, nsp.value) == (want_dp, want_sp), (r, ndp.value, nsp.value)
        tot_dp += ndp.value
        tot_sp += nsp.value
    assert tot_dp == lib.mt_dp_tiles(p, t, mode) and tot_sp == lib.mt_sp_tiles(p, t, mode)


def test_schedule_orders_every_step():
    for p in (1, 2, 5):
        acts = schedule(p)
        panels = [a[1] for a in acts if a[0] == "panel"]
        assert panels == list(range(p))
        # every update of step k comes after panel k's broadcast and covers k+1..p-1 once
        for k in range(p - 1):
            b = acts.index(("bcast", k))
            ups = [a for a in acts if a[0] == "update" and a[1] == k]
            cols = sorted(j for a in ups for j in range(a[2], a[3]))
            assert cols == list(range(k + 1, p))
            assert all(acts.index(a) > b for a in ups)
        # lookahead: panel k+1 is issued before the bulk update of step k
        for k in range(p - 1):
            assert acts.index(("panel", k + 1)) < acts.index(("update", k, k + 2, p))


# ------------------------------------------------------------ gloo protocol
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class NumpyRank:
    """Test-only tile backend: one rank's owned columns, the oracle's BLAS calls."""

    def __init__(self, tiles, n, nb, mode, t, rank, world):
        self.p = -(-n // nb)
        self.nb, self.mode, self.t, self.rank, self.world = nb, mode, t, rank, world
        self.dp, self.sp = {}, {}
        for (i, j), a in tiles.items():
            if owner(j, world) != rank:
                continue
            (self.dp if a.dtype == np.float64 else self.sp)[(i, j)] = np.array(a, order="F")
        self.panel = {}  # k -> {i: (dp, sp)}

    def do_panel(self, k):
        p, t, mp_ = self.p, self.t, self.mode == "mp"
        c, info = LP.dpotrf(self.dp[(k, k)], lower=1, clean=0, overwrite_a=1)
        if info > 0:
            raise O.NotSPD(k * self.nb + info - 1)
        self.dp[(k, k)] = c
        sp_diag = O.narrow(c) if (mp_ and k + t <= p - 1) else None
        rows = {}
        for i in range(k + 1, p):
            if self.mode == "dst" and i - k >= t:
                continue
            if i - k < t:
                x = B.dtrsm(1.0, c, self.dp[(i, k)], side=1, lower=1, trans_a=1, diag=0)
                self.dp[(i, k)] = x
                rows[i] = (x, O.narrow(x) if (mp_ and i + t <= p - 1) else None)
            else:
                s = B.strsm(1.0, sp_diag, self.sp[(i, k)], side=1, lower=1, trans_a=1, diag=0)
                self.sp[(i, k)] = s
                rows[i] = (O.widen(s), s)
        self.panel[k] = rows

    def do_update(self, k, jlo, jhi):
        rows, p, t = self.panel[k], self.p, self.t
        for j in range(jlo, jhi):
            if owner(j, self.world) != self.rank or j not in rows:
                continue
            self.dp[(j, j)] = B.dsyrk(-1.0, rows[j][0], beta=1.0, c=self.dp[(j, j)], trans=0,
                                      lower=1)
            for i in range(j + 1, p):
                if i not in rows or (self.mode == "dst" and i - j >= t):
                    continue
                if i - j < t:
                    self.dp[(i, j)] = B.dgemm(-1.0, rows[i][0], rows[j][0], beta=1.0,
                                              c=self.dp[(i, j)], trans_b=1)
                else:
                    self.sp[(i, j)] = B.sgemm(-1.0, rows[i][1], rows[j][1], beta=1.0,
                                              c=self.sp[(i, j)], trans_b=1)


def _worker(rank, world, port, n, nb, mode, t, queue):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "config1.npz"))
    locs, z = g["locs"][:n], g["z"][:n]
    tiles = O.assemble(locs, (1.0, 0.1, 0.5), nb, mode, t)
    R = NumpyRank(tiles, n, nb, mode, t, rank, world)
    for act in schedule(R.p):
        if act[0] == "panel":
            if owner(act[1], world) == rank:
                R.do_panel(act[1])
        elif act[0] == "bcast":
            k = act[1]
            box = [R.panel.get(k)]
            dist.broadcast_object_list(box, src=owner(k, world))
            R.panel[k] = box[0]
        else:
            R.do_update(*act[1:])
    # logdet: per-tile partials, one non-zero contributor each, fixed-order sum
    part = np.zeros(R.p)
    for k in range(R.p):
        if owner(k, world) == rank:
            part[k] = float(np.sum(np.log(np.diagonal(R.dp[(k, k)]))))
    box = [None] * world
    dist.all_gather_object(box, part)
    tot = 0.0
    for v in np.sum(box, axis=0).tolist():  # plain left-to-right (builtin sum() is compensated)
        tot += v
    ld = 2.0 * tot
    queue.put((rank, {k: v for k, v in R.dp.items()}, {k: v for k, v in R.sp.items()}, ld))
    dist.destroy_process_group()


@pytest.mark.parametrize("mode,t", [("mp", 2), ("dp", None), ("mp", 1)])
def test_gloo_protocol_bitwise_equals_single_process(mode, t):
    n, nb, world = 1024, 128, 2
    p = n // nb
    t = p if t is None else t
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, nb, mode, t, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "config1.npz"))
    ref = O.cholesky(O.assemble(g["locs"][:n], (1.0, 0.1, 0.5), nb, mode, t), n, nb, mode, t)
    seen = set()
    for rank, dp, sp, ld in res:
        for key, a in dp.items():
            if mode == "mp" and key[0] - key[1] >= t:
                continue  # off-band tiles hold FP32 payloads (checked via sp)
            assert np.array_equal(a, ref[key][0]), (rank, key)
            seen.add(key)
        for key, a in sp.items():
            assert np.array_equal(a, ref[key][1]), (rank, key)
            seen.add(key)
        assert ld == O.logdet(ref, p)
    assert seen == set(ref)
