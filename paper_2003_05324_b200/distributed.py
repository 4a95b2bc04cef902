"""Multi-GPU likelihood evaluation: one process per GPU, NCCL panel broadcast.

Layout: tile-column-cyclic (the 1 x g case of 2D block-cyclic): rank r stores
tile columns j = r, r + g, r + 2g, ... in local pools (storage scales as 1/g,
so full-DP N = 262144 fits on >= 2 B200s).  Step k of the right-looking
factorization (factor.py:44-80) becomes, with lookahead 1 on two streams:

    owner(k+1), panel stream:  update(k -> column k+1), POTRF(k+1), TRSM(k+1)
    everyone, panel stream:    broadcast panel k+1 from owner(k+1) (NCCL)
    everyone, caller stream:   update(k -> owned columns k+2 .. p-1), which
                               overlaps the panel chain and the broadcast and
                               yields SMs to the panel kernels on request

A panel is broadcast as the TF32 hi/lo split of its FP32 operands (rows
k+1..p-1, what the tcgen05 update reads) plus its FP64 band rows (what the
DMMA update reads), straight into every rank's panel ring.  Every tile
receives the same updates in the same order from the same kernels as on one
GPU, so factor, logdet and quad are bitwise identical for any rank count
(tests/test_gpu_distributed.py).  logdet: per-diagonal-tile partials
all-reduced (each entry has one non-zero contributor, so the sum is exact)
then summed in fixed order; quad: forward sweep with the vector broadcast
from each column owner, then the single-GPU reduction kernel.
"""

import ctypes
import math

from . import _lib
from .factor import FactorizationError
from .tilestore import PrecisionOverflowError, TileMatrix

LOG_2PI = math.log(2.0 * math.pi)


def owner(j, world):
    """Rank that stores tile column j."""
    return j % world


def schedule(p):
    """Rank-independent action order of the distributed factorization (what
    DistributedEvaluator.factor issues, the first three of each step on the
    panel stream, the last on the caller stream).

    ("panel", k)            POTRF(k) + TRSM(k), executed by owner(k)
    ("bcast", k)            panel k broadcast from owner(k) to every rank
    ("update", k, jlo, jhi) step-k updates of each rank's owned columns in [jlo, jhi)
    """
    acts = [("panel", 0), ("bcast", 0)]
    for k in range(p - 1):
        acts += [("update", k, k + 1, k + 2), ("panel", k + 1), ("bcast", k + 1),
                 ("update", k, k + 2, p)]
    return acts


def panel_slices(m, k):
    """(tensor view, description) pairs holding panel k in a rank's panel rings."""
    p, te, t = m.p, m.nb * m.nb, m.policy.diag_thick
    out = []
    if m.split is not None and k + 1 < p:
        base = ((k & 1) * p + k + 1) * 2 * te
        out.append(m.split[base: ((k & 1) * p + p) * 2 * te])
    rows = min(p, k + t) - (k + 1)  # band rows k+1 .. k+t-1
    if rows > 0:
        base = ((k & 1) * t + 1) * te
        out.append(m.dpanel[base: base + rows * te])
    return out


class DistributedEvaluator:
    """Likelihood evaluations of one dataset split over the ranks of `group`
    (torch.distributed, NCCL on GPUs; gloo works for 1-GPU testing)."""

    def __init__(self, assembler, policy, group=None):
        torch = _lib.require_cuda()
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.asm = assembler
        self.matrix = TileMatrix(assembler.n, assembler.nb, policy,
                                 col_stride=self.world, col_offset=self.rank)
        m = self.matrix
        if self.world > 1 and (m.nb % 256 or (m.policy.mode.value == "mp" and m.split is None)):
            raise ValueError("the multi-GPU path needs nb % 256 == 0 (tcgen05 split panels)")
        dev = m.device
        npad = m.p * m.nb
        self.x = torch.empty(npad, dtype=torch.float64, device=dev)
        self.partial = torch.empty(m.p, dtype=torch.float64, device=dev)
        self.work = torch.empty(2048, dtype=torch.float64, device=dev)
        self.out = torch.empty(1, dtype=torch.float64, device=dev)
        self.flag = torch.empty(3, dtype=torch.int64, device=dev)
        self.pan = torch.cuda.Stream(device=dev, priority=-1)
        self.yield_sms = 32  # SMs the bulk update releases to the owner's panel kernels

    # -- pieces -------------------------------------------------------------
    def _bcast(self, k, async_op):
        src = owner(k, self.world)
        return [self.dist.broadcast(v, src=src, group=self.group, async_op=async_op)
                for v in panel_slices(self.matrix, k)]

    def factor(self):
        """The step loop with lookahead 1 on two streams (the single-GPU
        schedule of csrc/api.cu, with the broadcast in the panel chain):

          panel stream (high priority): update(k -> column k+1) on its owner,
                         POTRF+TRSM(k+1) on its owner, broadcast of panel k+1
          caller stream: update(k -> owned columns k+2 ..), which yields SMs
                         to the owner's panel kernels on request

        The panel stream waits for the caller's step k-1 before touching the
        panel ring slot of k+1 (= slot of k-1) and column k+1."""
        torch = _lib.require_cuda()
        m, lib = self.matrix, _lib.load()
        d = ctypes.byref(m.desc)
        main, pan = torch.cuda.current_stream(), self.pan
        hm, hp = ctypes.c_void_p(main.cuda_stream), ctypes.c_void_p(pan.cuda_stream)
        mine = lambda k: owner(k, self.world) == self.rank  # noqa: E731
        bc = {}

        def panel(k):  # on the panel stream
            if mine(k):
                _lib.check(lib.mt_yield_request(self.yield_sms, hp), "mt_yield_request")
                _lib.check(lib.mt_panel(d, k, hp), "mt_panel")
                _lib.check(lib.mt_yield_request(0, hp), "mt_yield_request")
            if self.world > 1:
                with torch.cuda.stream(pan):
                    bc[k] = self._bcast(k, async_op=True)

        def received(k):  # the current stream waits for panel k's broadcast
            for h in bc.get(k, []):
                h.wait()

        pan.wait_stream(main)  # generation of the local tiles
        panel(0)
        step_done = None
        for k in range(m.p - 1):
            with torch.cuda.stream(pan):
                if step_done is not None:
                    pan.wait_event(step_done)  # step k-1 applied everywhere on this rank
                if mine(k + 1):
                    received(k)
                    _lib.check(lib.mt_update(d, k, k + 1, k + 2, hp), "mt_update")
            panel(k + 1)
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
        m, lib, st = self.matrix, _lib.load(), _lib.stream_handle()
        self.x.copy_(self.asm.d_z)
        nb = m.nb
        for i in range(m.p):
            if owner(i, self.world) == self.rank:
                _lib.check(lib.mt_fwd_step(ctypes.byref(m.desc), i, _lib.ptr(self.x), st),
                           "mt_fwd_step")
            if self.world > 1:
                self.dist.broadcast(self.x[i * nb:], src=owner(i, self.world), group=self.group)
        _lib.check(lib.mt_sumsq(_lib.ptr(self.x), self.x.numel(), _lib.ptr(self.work),
                                _lib.ptr(self.out), st), "mt_sumsq")
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


def loglik_distributed(dataset, params, nb, policy, group=None):
    """Distributed counterpart of mle.loglik (mle.py:89-99); call on every rank."""
    from .mle import LikelihoodEval
    from .tilestore import TileAssembler
    ev = DistributedEvaluator(TileAssembler(dataset, nb), policy, group)
    ld, quad = ev(params)
    return LikelihoodEval(-0.5 * (dataset.n * LOG_2PI + ld + quad), ld, quad)
