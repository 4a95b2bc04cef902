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
from paper_2003_05324_b200.distributed import (owner, panel_bcast_plan, ring_geometry, ring_pos,
                                                  schedule, tile_owner)


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
    """Test-only tile backend: one rank's tiles of a P x Q grid, the oracle's
    BLAS calls, and the same broadcast plan as DistributedEvaluator."""

    def __init__(self, tiles, n, nb, mode, t, rank, P, Q):
        self.p = -(-n // nb)
        self.nb, self.mode, self.t = nb, mode, t
        self.rank, self.P, self.Q = rank, P, Q
        self.pr, self.pc = divmod(rank, Q)
        self.dp, self.sp = {}, {}
        for (i, j), a in tiles.items():
            if tile_owner(i, j, P, Q) != rank:
                continue
            (self.dp if a.dtype == np.float64 else self.sp)[(i, j)] = np.array(a, order="F")
        self.panel = {}  # k -> {i: (dp or None, sp or None)}
        self.diag = {}

    def mine(self, i, j):
        return tile_owner(i, j, self.P, self.Q) == self.rank

    def do_factor(self, k):
        c, info = LP.dpotrf(self.dp[(k, k)], lower=1, clean=0, overwrite_a=1)
        if info > 0:
            raise O.NotSPD(k * self.nb + info - 1)
        self.dp[(k, k)] = c
        p, t = self.p, self.t
        self.diag[k] = (c, O.narrow(c) if (self.mode == "mp" and k + t <= p - 1) else None)

    def do_solve(self, k):
        p, t, mp_ = self.p, self.t, self.mode == "mp"
        c, sp_diag = self.diag[k]
        rows = self.panel.setdefault(k, {})
        for i in range(k + 1, p):
            if not self.mine(i, k) or (self.mode == "dst" and i - k >= t):
                continue
            if i - k < t:
                x = B.dtrsm(1.0, c, self.dp[(i, k)], side=1, lower=1, trans_a=1, diag=0)
                self.dp[(i, k)] = x
                rows[i] = (x, O.narrow(x) if (mp_ and i + t <= p - 1) else None)
            else:
                s = B.strsm(1.0, sp_diag, self.sp[(i, k)], side=1, lower=1, trans_a=1, diag=0)
                self.sp[(i, k)] = s
                rows[i] = (None, s)  # FP32 rows travel without an FP64 copy (split only)

    def row(self, k, i):
        """(FP64 view, FP32 payload) of panel row i; the FP64 view of an FP32 row
        is its exact widening (the DMMA update widens the split on load)."""
        d, s = self.panel[k][i]
        return (d if d is not None else O.widen(s)), s

    def do_update(self, k, jlo, jhi):
        p, t, rows = self.p, self.t, self.panel[k]
        for j in range(jlo, jhi):
            if j % self.Q != self.pc or j not in rows and not any(
                    self.mine(i, j) for i in range(j, p)):
                continue
            if self.mine(j, j) and j in rows:
                self.dp[(j, j)] = B.dsyrk(-1.0, self.row(k, j)[0], beta=1.0, c=self.dp[(j, j)],
                                          trans=0, lower=1)
            for i in range(j + 1, p):
                if not self.mine(i, j) or i not in rows or j not in rows:
                    continue
                if self.mode == "dst" and i - j >= t:
                    continue
                if i - j < t:
                    self.dp[(i, j)] = B.dgemm(-1.0, self.row(k, i)[0], self.row(k, j)[0], beta=1.0,
                                              c=self.dp[(i, j)], trans_b=1)
                else:
                    self.sp[(i, j)] = B.sgemm(-1.0, rows[i][1], rows[j][1], beta=1.0,
                                              c=self.sp[(i, j)], trans_b=1)


def _group_of(groups, idx):
    return groups[idx] if groups else None


def _worker(rank, world, P, Q, port, n, nb, mode, t, queue):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows_g = [dist.new_group([r * Q + c for c in range(Q)]) for r in range(P)] if P > 1 and Q > 1 else []
    cols_g = [dist.new_group([r * Q + c for r in range(P)]) for c in range(Q)] if P > 1 and Q > 1 else []
    row_of = lambda r: rows_g[r] if rows_g else None  # noqa: E731  (1 x Q: the world)
    col_of = lambda c: cols_g[c] if cols_g else None  # noqa: E731  (P x 1: the world)
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "config1.npz"))
    locs, z = g["locs"][:n], g["z"][:n]
    tiles = O.assemble(locs, (1.0, 0.1, 0.5), nb, mode, t)
    R = NumpyRank(tiles, n, nb, mode, t, rank, P, Q)
    p = R.p
    L, _, _ = ring_geometry(p, P, Q)

    def panel(k):
        if k % Q == R.pc:
            if R.mine(k, k):
                R.do_factor(k)
            if P > 1:
                box = [R.diag.get(k)]
                dist.broadcast_object_list(box, src=(k % P) * Q + R.pc, group=col_of(R.pc))
                R.diag[k] = box[0]
            R.do_solve(k)
        rows = R.panel.setdefault(k, {})
        for stage, grp, root, b, m0, m1, mb1 in panel_bcast_plan(k, p, P, Q, t):
            if (stage == "row" and grp != R.pr) or (stage == "col" and grp != R.pc):
                continue
            idx = [b + L * m for m in range(m0, m1 + 1)]
            band = {b + L * m for m in range(m0, mb1 + 1)}
            box = [None]
            if rank == root:
                # FP64 rows only for the band (m <= mb1), as the GPU's ring slices
                box = [{i: (rows[i][0] if i in band else None, rows[i][1]) for i in idx
                        if i in rows}]
            dist.broadcast_object_list(box, src=root, group=row_of(grp) if stage == "row" else col_of(grp))
            for i, (d, s_) in box[0].items():
                rows[i] = (d, s_)

    panel(0)
    for k in range(p - 1):
        R.do_update(k, k + 1, k + 2)
        panel(k + 1)
        if k + 2 < p:
            R.do_update(k, k + 2, p)
    # logdet: per-tile partials, one non-zero contributor each, fixed-order sum
    part = np.zeros(p)
    for k in range(p):
        if R.mine(k, k):
            part[k] = float(np.sum(np.log(np.diagonal(R.dp[(k, k)]))))
    box = [None] * world
    dist.all_gather_object(box, part)
    tot = 0.0
    for v in np.sum(box, axis=0).tolist():  # plain left-to-right (builtin sum() is compensated)
        tot += v
    ld = 2.0 * tot
    queue.put((rank, {k: v for k, v in R.dp.items()}, {k: v for k, v in R.sp.items()}, ld))
    dist.destroy_process_group()


@pytest.mark.parametrize("P,Q,mode,t", [(1, 2, "mp", 2), (1, 2, "dp", None), (2, 2, "mp", 2),
                                        (2, 2, "dp", None), (2, 1, "mp", 1), (2, 2, "mp", 3)])
def test_gloo_protocol_bitwise_equals_single_process(P, Q, mode, t):
    n, nb = 1024, 128
    world = P * Q
    p = n // nb
    t = p if t is None else t
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, P, Q, port, n, nb, mode, t, q))
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


@pytest.mark.parametrize("P,Q", [(1, 1), (1, 4), (2, 2), (2, 4), (4, 2), (2, 3), (3, 2)])
@pytest.mark.parametrize("p,t", [(16, 2), (17, 5), (9, 9)])
def test_panel_plan_reaches_every_consumer(P, Q, p, t):
    """Every rank receives (or owns) exactly the panel rows its tiles consume,
    and each broadcast's root holds the rows it sends; the ring positions are
    the library's (mt_ring_pos) and form a bijection onto the ring."""
    lib = _lib.load()
    L, rq, pring = ring_geometry(p, P, Q)
    pos = [ring_pos(i, p, P, Q) for i in range(p)]
    assert pos == [lib.mt_ring_pos(p, P, Q, i) for i in range(p)]
    assert len(set(pos)) == p and max(pos) < pring
    assert 2 * pring == lib.mt_dpanel_tiles_ex(p, P, Q)
    for k in range(p - 1):
        have = {r: {i for i in range(k + 1, p) if tile_owner(i, k, P, Q) == r}
                for r in range(P * Q)}
        for stage, grp, root, b, m0, m1, mb1 in panel_bcast_plan(k, p, P, Q, t):
            rows = {b + L * m for m in range(m0, m1 + 1)}
            assert rows and all(k < i < p for i in rows)
            assert rows <= have[root], (stage, grp, root, b)
            members = ([grp * Q + c for c in range(Q)] if stage == "row"
                       else [r * Q + grp for r in range(P)])
            assert root in members
            for r in members:
                have[r] |= rows
            # FP64 rows: the band rows i - k < t of the block
            assert {b + L * m for m in range(m0, mb1 + 1)} == {i for i in rows if i - k < t}
        for r in range(P * Q):
            pr_, pc_ = divmod(r, Q)
            need = set()
            for j in range(k + 1, p):
                for i in range(j, p):
                    if i % P == pr_ and j % Q == pc_:
                        need |= {i, j}
            assert need <= have[r], (k, r, sorted(need - have[r]))


@pytest.mark.parametrize("P,Q", [(1, 3), (2, 2), (2, 3), (4, 2)])
@pytest.mark.parametrize("p,t,mode", [(16, 2, 1), (16, 16, 0), (9, 3, 1), (7, 1, 1), (12, 4, 2)])
def test_2d_local_layout_matches_bruteforce(P, Q, p, t, mode):
    lib = _lib.load()
    tot_dp = tot_sp = 0
    for r in range(P):
        for c in range(Q):
            ndp, nsp = ctypes.c_int64(), ctypes.c_int64()
            lib.mt_local_tiles_ex(p, t, mode, P, r, Q, c, ctypes.byref(ndp), ctypes.byref(nsp))
            tt = t if mode else p
            want_dp = sum(1 for j in range(c, p, Q) for i in range(j, min(j + tt, p)) if i % P == r)
            want_sp = (sum(1 for j in range(c, p, Q) for i in range(j + t, p) if i % P == r)
                       if mode == 1 else 0)
            assert (ndp.value, nsp.value) == (want_dp, want_sp), (r, c)
            tot_dp += ndp.value
            tot_sp += nsp.value
    assert tot_dp == lib.mt_dp_tiles(p, t, mode) and tot_sp == lib.mt_sp_tiles(p, t, mode)
