"""GPU: the multi-GPU path (distributed.DistributedEvaluator) end to end.

The gpurun box has one B200, so the ranks share cuda:0 and talk over gloo
(NCCL refuses two ranks on one device); the CUDA kernels, local pools,
panel rings and the step schedule are the ones a multi-GPU NCCL run uses.
Factor tiles, logdet and quad must be bitwise identical to one GPU.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data(n):
    from conftest import load_golden
    g = load_golden("config1")
    return g["locs"][:n], g["z"][:n]


def _policy(mt, tag):
    if tag == "dp":
        return mt.PrecisionPolicy.dp()
    mode, t = tag.split(":")
    return getattr(mt.PrecisionPolicy, mode)(diag_thick=int(t))


def _worker(rank, world, port, n, nb, tag, queue, grid=None):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2003_05324_b200 as mt
    from paper_2003_05324_b200.distributed import DistributedEvaluator
    locs, z = _data(n)
    ds = mt.GeoDataset(locs, z)
    pol = _policy(mt, tag)
    ev = DistributedEvaluator(mt.TileAssembler(ds, nb), pol, grid=grid)
    try:
        ld, quad = ev(mt.MaternParams(1.0, 0.1, 0.5))
    except mt.FactorizationError as exc:  # (DST may be indefinite: same pivot everywhere)
        queue.put((rank, "npd", exc.index, None))
        dist.destroy_process_group()
        return
    tiles = {key: (t.dp, t.sp) for key, t in ev.matrix.tiles.items()}
    queue.put((rank, ld, quad, tiles))
    dist.destroy_process_group()


@pytest.mark.parametrize("tag,grid", [("mp:2", (1, 2)), ("dp", (1, 2)), ("mp:1", (1, 2)),
                                      ("mp:2", (2, 2)), ("dp", (2, 2)), ("mp:3", (2, 1)),
                                      ("mp:2", (2, 1)), ("dst:2", (2, 2))])
def test_ranks_bitwise_equal_single_gpu(gpu, tag, grid):
    """1 x 2, 2 x 1 and 2 x 2 process grids (2D block-cyclic tiles, row and
    column sub-communicators): factor, logdet and quad bitwise equal to one GPU."""
    import sys
    import torch.multiprocessing as mp
    import paper_2003_05324_b200 as mt
    n, nb = 2048, 256
    world = grid[0] * grid[1]
    here = os.path.dirname(os.path.abspath(__file__))
    if here not in sys.path:
        sys.path.insert(0, here)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, nb, tag, q, grid))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    locs, z = _data(n)
    pol = _policy(mt, tag)
    ev = mt.Evaluator(mt.TileAssembler(mt.GeoDataset(locs, z), nb), pol, lookahead=1)
    try:
        ld1, q1 = ev(mt.MaternParams(1.0, 0.1, 0.5))
    except mt.FactorizationError as exc:
        assert all(r[1] == "npd" and r[2] == exc.index for r in res), (exc.index, res)
        return
    ref = ev.matrix.tiles
    seen = set()
    for rank, ld, quad, tiles in res:
        assert ld == ld1 and quad == q1, (rank, ld, ld1, quad, q1)
        for key, (dp, sp) in tiles.items():
            r = ref[key]
            if sp is not None:
                assert np.array_equal(sp, r.sp), (rank, key)
            else:
                assert np.array_equal(dp, r.dp), (rank, key)
            assert key not in seen, key  # every tile stored by exactly one rank
            seen.add(key)
    assert seen == set(ref)
