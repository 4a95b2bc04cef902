"""Multi-GPU likelihood evaluation: one process per GPU, 2D block-cyclic tiles.

Layout (north_star): a P x Q process grid, rank = r * Q + c;
rank (r, c) stores the tiles (i, j) with i = r (mod P), j = c (mod Q) in
local pools (storage ~1/(PQ) of the matrix: full DP at N = 262144 fits on
2 B200s).  The reference's task DAG (factor.py:44-80) becomes, per step k:

  owner of (k, k):        POTRF(k) [+ W = L_kk^{-1} for the tensor-core TRSM]
  process column k%Q:     L_kk, its 32x32 inverses and W broadcast down the
                          column (P > 1), then TRSM(k) of each rank's rows
  every rank:             panel k's rows broadcast along process rows (each row
                          operand A_ik reaches the ranks of row i%P), then down
                          process columns (each column operand A_jk reaches the
                          ranks of column j%Q)
  every rank:             trailing update of its own tiles

with lookahead 1 on two streams: the ranks of process column (k+1)%Q update
tile column k+1 and factor panel k+1 on a high-priority panel stream while
every rank applies step k to the rest of its tiles (yielding SMs to the panel
kernels on request).  Panel rows travel as the TF32 hi/lo split of their FP32
payload (what the tcgen05 update reads) plus FP64 rows for the band, in
"ring order": tile row i sits at (i mod L) * ceil(p/L) + i // L, L = lcm(P, Q)
(L = 1 on a 1 x Q grid), so every broadcast is one contiguous slice of a
block of rows i = b (mod L).  Every tile receives the same updates in the
same order from the same kernels as on one GPU, so the factor, logdet and
quad are bitwise identical for any grid (tests/test_gpu_distributed.py,
tests/test_distributed_cpu.py).  logdet: per-diagonal-tile partials,
all-reduced (one non-zero contributor each: exact) and summed in fixed order;
quad: the forward sweep y = L^{-1} z fused into the schedule, step i on the
panel stream right after panel i -- TRSV on the owner of (i, i), y_i down
process column i%Q, GEMV of each rank's rows, the updated x along process
rows -- then y gathered exactly and reduced as on one GPU.
"""

import ctypes
import math

from . import _lib
from .factor import FactorizationError
from .tilestore import PrecisionOverflowError, TileMatrix

LOG_2PI = math.log(2.0 * math.pi)
_GROUPS = {}  # (member ranks, P, Q) -> (row groups, column groups)


# --------------------------------------------------------------- grid plan
def grid_shape(world, grid=None):
    """(P, Q) of the process grid: `grid` if given, else 1 x world."""
    if grid is None:
        return 1, world
    P, Q = int(grid[0]), int(grid[1])
    if P < 1 or Q < 1 or P * Q != world:
        raise ValueError(f"process grid {P}x{Q} does not match {world} ranks")
    return P, Q


def owner(j, world):
    """Rank that stores tile column j on a 1 x world grid."""
    return j % world


def tile_owner(i, j, P, Q):
    """Rank storing tile (i, j) on a P x Q grid."""
    return (i % P) * Q + (j % Q)


def ring_geometry(p, P, Q):
    """(L, rows per block, ring length) of the panel ring order (csrc/mt_grid.cuh)."""
    L = 1 if P == 1 else P // math.gcd(P, Q) * Q
    rq = -(-p // L)
    return L, rq, L * rq


def ring_pos(i, p, P, Q):
    L, rq, _ = ring_geometry(p, P, Q)
    return i if L == 1 else (i % L) * rq + i // L


def panel_bcast_plan(k, p, P, Q, t):
    """Broadcasts that distribute panel k, in issue order (the same on every rank).

    Each entry is (stage, group, root, b, m0, m1, mb1): stage "row" runs in
    process row `group` (root = the rank of column k%Q there), stage "col" in
    process column `group` (root = the rank of row b%P there); block b holds
    rows i = b + L*m, the broadcast covers m in [m0, m1] of the split ring and
    m in [m0, mb1] of the FP64 ring (rows with i - k < t; mb1 < m0: none)."""
    L, rq, _ = ring_geometry(p, P, Q)
    out = []

    def rng(b):
        m0 = 0 if b > k else (k - b) // L + 1
        m1 = (p - 1 - b) // L
        mb1 = (min(k + t, p) - 1 - b) // L if min(k + t, p) - 1 >= b else -1
        return m0, m1, mb1

    if Q > 1:
        for b in range(L):
            m0, m1, mb1 = rng(b)
            if m0 <= m1:
                r = b % P
                out.append(("row", r, r * Q + k % Q, b, m0, m1, mb1))
    if P > 1:
        for b in range(L):
            m0, m1, mb1 = rng(b)
            if m0 <= m1:
                c = b % Q
                out.append(("col", c, (b % P) * Q + c, b, m0, m1, mb1))
    return out


def schedule(p):
    """Rank-independent action order of the 1 x g factorization (panel = POTRF +
    TRSM on the column owner, bcast = its panel to every rank, update = step-k
    updates of each rank's columns in [jlo, jhi))."""
    acts = [("panel", 0), ("bcast", 0)]
    for k in range(p - 1):
        acts += [("update", k, k + 1, k + 2), ("panel", k + 1), ("bcast", k + 1),
                 ("update", k, k + 2, p)]
    return acts


# ------------------------------------------------------------- evaluator
class DistributedEvaluator:
    """Likelihood evaluations of one dataset split over the ranks of `group`
    (torch.distributed, NCCL on GPUs; gloo works for 1-GPU testing) on a
    P x Q process grid (`grid`, default 1 x world)."""

    def __init__(self, assembler, policy, group=None, grid=None):
        torch = _lib.require_cuda()
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.P, self.Q = grid_shape(self.world, grid)
        self.pr, self.pc = divmod(self.rank, self.Q)
        members = (dist.get_process_group_ranks(group) if group is not None
                   else list(range(self.world)))
        self.members = members
        # sub-communicators: every rank creates every group, in the same order;
        # cached per (members, grid) so repeated evaluators (loglik_distributed,
        # fit loops) do not re-create NCCL communicators
        self.row_groups, self.col_groups = [], []
        if self.P > 1 and self.Q > 1:
            key = (tuple(members), self.P, self.Q)
            if key not in _GROUPS:
                _GROUPS[key] = (
                    [dist.new_group([members[r * self.Q + c] for c in range(self.Q)])
                     for r in range(self.P)],
                    [dist.new_group([members[r * self.Q + c] for r in range(self.P)])
                     for c in range(self.Q)])
            self.row_groups, self.col_groups = _GROUPS[key]
        elif self.Q > 1:
            self.row_groups = [group]
        elif self.P > 1:
            self.col_groups = [group]
        self.asm = assembler
        self.matrix = TileMatrix(assembler.n, assembler.nb, policy, col_stride=self.Q,
                                 col_offset=self.pc, row_stride=self.P, row_offset=self.pr)
        m = self.matrix
        if self.world > 1 and (m.nb % 256 or (m.policy.mode.value == "mp" and m.split is None)):
            raise ValueError("the multi-GPU path needs nb % 256 == 0 (tcgen05 split panels)")
        dev = m.device
        npad = m.p * m.nb
        self.x = torch.empty(npad, dtype=torch.float64, device=dev)
        self.y = torch.empty(npad, dtype=torch.float64, device=dev)
        self.partial = torch.empty(m.p, dtype=torch.float64, device=dev)
        self.work = torch.empty(2048, dtype=torch.float64, device=dev)
        self.out = torch.empty(1, dtype=torch.float64, device=dev)
        self.flag = torch.empty(3, dtype=torch.int64, device=dev)
        self.pan = torch.cuda.Stream(device=dev, priority=-1)
        self.yield_sms = 32  # SMs the bulk update releases to the panel kernels

    # -- helpers ------------------------------------------------------------
    def _grank(self, r):
        """Global rank (torch.distributed) of grid rank r."""
        return self.members[r]

    def _mine_col(self, k):
        return k % self.Q == self.pc

    def _mine_diag(self, k):
        return k % self.P == self.pr and k % self.Q == self.pc

    def _bcast(self, tensor, root, groups, index, async_op):
        """Broadcast from grid rank `root` inside groups[index] (the whole
        group when the grid is one row or one column)."""
        return self.dist.broadcast(tensor, src=self._grank(root), group=groups[index],
                                   async_op=async_op)

    def _diag_bcast(self, k):
        """L_kk (FP64 ring row k), its 32x32 inverses and W's split, down
        process column k%Q from the owner of (k, k)."""
        m, lib = self.matrix, _lib.load()
        reg = (ctypes.c_int64 * 6)()
        _lib.check(lib.mt_diag_regions(ctypes.byref(m.desc), k, reg), "mt_diag_regions")
        root = (k % self.P) * self.Q + self.pc
        views = [m.dpanel[reg[0]: reg[0] + reg[1]], m.scratch[reg[2]: reg[2] + reg[3]]]
        if reg[5] > 0:
            views.append(m.split[reg[4]: reg[4] + reg[5]])
        for v in views:
            if v.numel():
                self._bcast(v, root, self.col_groups, 0 if self.Q == 1 else self.pc, False)

    def _panel_bcast(self, k):
        """Distribute panel k (panel_bcast_plan); returns the async handles."""
        m = self.matrix
        p, te, t = m.p, m.nb * m.nb, m.policy.diag_thick
        L, rq, pring = ring_geometry(p, self.P, self.Q)
        base = (k & 1) * pring
        hs = []
        row_done = False
        for stage, grp, root, b, m0, m1, mb1 in panel_bcast_plan(k, p, self.P, self.Q, t):
            if stage == "col" and not row_done:
                # a column-stage root forwards rows it received in the row stage:
                # collectives of different communicators are not ordered with
                # each other, so the current stream waits for the row stage here
                for h in hs:
                    h.wait()
                row_done = True
            if stage == "row":
                if grp != self.pr:
                    continue
                groups, index = self.row_groups, (0 if self.P == 1 else grp)
            else:
                if grp != self.pc:
                    continue
                groups, index = self.col_groups, (0 if self.Q == 1 else grp)
            r0 = base + b * rq
            if m.split is not None:
                v = m.split[(r0 + m0) * 2 * te: (r0 + m1 + 1) * 2 * te]
                hs.append(self._bcast(v, root, groups, index, True))
            if mb1 >= m0:
                v = m.dpanel[(r0 + m0) * te: (r0 + mb1 + 1) * te]
                hs.append(self._bcast(v, root, groups, index, True))
        return hs

    # -- factorization --------------------------------------------------------
    def factor(self):
        """The step loop with lookahead 1 on two streams (the single-GPU
        schedule of csrc/api.cu with the collectives in the panel chain):

          panel stream (high priority): update(k -> column k+1) on the ranks of
                         its process column, POTRF(k+1) on the owner of
                         (k+1, k+1), the column broadcast of L, TRSM(k+1), the
                         row/column broadcasts of panel k+1
          caller stream: update(k -> this rank's columns k+2 ..), which yields
                         SMs to the panel kernels on request

        The panel stream waits for the caller's step k-1 before touching the
        ring slot of k+1 (= slot of k-1) and column k+1."""
        torch = _lib.require_cuda()
        m, lib = self.matrix, _lib.load()
        d = ctypes.byref(m.desc)
        main, pan = torch.cuda.current_stream(), self.pan
        hm, hp = ctypes.c_void_p(main.cuda_stream), ctypes.c_void_p(pan.cuda_stream)
        multi = self.world > 1
        bc = {}
        x, nb, P, Q = self.x, m.nb, self.P, self.Q
        x.copy_(self.asm.d_z)  # the forward sweep of quad runs fused into the schedule

        def fwd(i):  # forward-sweep step i on the panel stream, right after panel i
            with torch.cuda.stream(pan):
                if self._mine_diag(i):
                    _lib.check(lib.mt_fwd_step_ex(d, i, 1, _lib.ptr(x), hp), "mt_fwd_step_ex")
                if self._mine_col(i):
                    if P > 1:
                        self._bcast(x[i * nb:(i + 1) * nb], (i % P) * Q + self.pc,
                                    self.col_groups, 0 if Q == 1 else self.pc, False)
                    _lib.check(lib.mt_fwd_step_ex(d, i, 2, _lib.ptr(x), hp), "mt_fwd_step_ex")
                if Q > 1 and i + 1 < m.p:
                    self._bcast(x[(i + 1) * nb:], self.pr * Q + i % Q, self.row_groups,
                                0 if P == 1 else self.pr, False)

        def panel(k):  # on the panel stream
            with torch.cuda.stream(pan):
                if self._mine_col(k):
                    _lib.check(lib.mt_yield_request(self.yield_sms, hp), "mt_yield_request")
                    if self._mine_diag(k):
                        _lib.check(lib.mt_panel_factor(d, k, hp), "mt_panel_factor")
                    if self.P > 1:
                        self._diag_bcast(k)
                    _lib.check(lib.mt_panel_solve(d, k, hp), "mt_panel_solve")
                    _lib.check(lib.mt_yield_request(0, hp), "mt_yield_request")
                if multi:
                    bc[k] = self._panel_bcast(k)

        def received(k):  # the current stream waits for panel k's broadcasts
            for h in bc.get(k, []):
                h.wait()

        pan.wait_stream(main)  # generation of the local tiles, x = z
        panel(0)
        fwd(0)
        step_done = None
        for k in range(m.p - 1):
            with torch.cuda.stream(pan):
                if step_done is not None:
                    pan.wait_event(step_done)  # step k-1 applied everywhere on this rank
                if self._mine_col(k + 1):
                    received(k)
                    _lib.check(lib.mt_update(d, k, k + 1, k + 2, hp), "mt_update")
            panel(k + 1)
            fwd(k + 1)
            received(k)
            bc.pop(k, None)
            if k + 2 < m.p:
                _lib.check(lib.mt_update_ex(d, k, k + 2, m.p, 1, hm), "mt_update_ex")
            step_done = main.record_event()
        main.wait_stream(pan)
        received(m.p - 1)
        bc.clear()
        m._touch()
        m.factored = True

    def status(self):
        """Agree on (first bad pivot, overflow count) across ranks."""
        bad, ov, _ = self.matrix.read_status()
        f = self.flag
        f[0] = bad if bad >= 0 else 2 ** 62
        f[1] = ov
        f[2] = 0
        if self.world > 1:
            self.dist.all_reduce(f[:1], op=self.dist.ReduceOp.MIN, group=self.group)
            self.dist.all_reduce(f[1:2], op=self.dist.ReduceOp.SUM, group=self.group)
        bad = int(f[0].item())
        return (bad if bad < 2 ** 62 else -1), int(f[1].item())

    def logdet(self):
        m, lib, st = self.matrix, _lib.load(), _lib.stream_handle()
        _lib.check(lib.mt_logdet_partials(ctypes.byref(m.desc), _lib.ptr(self.partial), st),
                   "mt_logdet_partials")
        if self.world > 1:
            self.dist.all_reduce(self.partial, group=self.group)
        tot = 0.0
        for v in self.partial.cpu().tolist():  # fixed order, as fixed_sum_kernel
            tot += v
        return 2.0 * tot

    def quad(self):
        """||L^{-1} z||^2 after factor(): the forward sweep ran inside the
        schedule (see the module docstring); y_i lives on the owner of (i, i),
        gathered exactly (one non-zero term per entry) and reduced in the
        single-GPU order."""
        m, lib, st = self.matrix, _lib.load(), _lib.stream_handle()
        nb, x, y = m.nb, self.x, self.y
        y.zero_()
        for i in range(m.p):
            if self._mine_diag(i):
                y[i * nb:(i + 1) * nb] = x[i * nb:(i + 1) * nb]
        if self.world > 1:
            self.dist.all_reduce(y, group=self.group)
        _lib.check(lib.mt_sumsq(_lib.ptr(y), y.numel(), _lib.ptr(self.work), _lib.ptr(self.out),
                                st), "mt_sumsq")
        return float(self.out.item())

    def __call__(self, params, chol_events=None):
        """(logdet, quad) of one evaluation; same values on every rank.
        chol_events: optional (start, end) CUDA events around the factorization."""
        m = self.matrix
        m.reset_status()
        m.factored = False
        self.asm.generate_into(m, params)
        if chol_events is not None:
            chol_events[0].record()
        self.factor()
        if chol_events is not None:
            chol_events[1].record()
        bad, ov = self.status()
        if ov:
            raise PrecisionOverflowError(f"{ov} value(s) exceed FP32 range during narrowing")
        if bad >= 0:
            raise FactorizationError(bad)
        return self.logdet(), self.quad()


def loglik_distributed(dataset, params, nb, policy, group=None, grid=None):
    """Distributed counterpart of mle.loglik (mle.py:89-99); call on every rank."""
    from .mle import LikelihoodEval
    from .tilestore import TileAssembler
    ev = DistributedEvaluator(TileAssembler(dataset, nb), policy, group, grid)
    ld, quad = ev(params)
    return LikelihoodEval(-0.5 * (dataset.n * LOG_2PI + ld + quad), ld, quad)
