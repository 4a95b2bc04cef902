"""2-rank gloo run of DistributedEvaluator on one GPU with stack dumps on hang (dev tool)."""
import faulthandler, os, socket, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np


def worker(rank, world, port, tag, ys):
    faulthandler.dump_traceback_later(40, exit=True)
    import torch, torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2003_05324_b200 as mt
    from paper_2003_05324_b200.distributed import DistributedEvaluator
    n, nb = 2048, 256
    locs = mt.generate_locations(n, seed=3)
    ds, _ = mt.morton_sort(mt.GeoDataset(locs, np.random.default_rng(1).standard_normal(n)))
    pol = mt.PrecisionPolicy.mp(diag_thick=2) if tag == "mp" else mt.PrecisionPolicy.dp()
    ev = DistributedEvaluator(mt.TileAssembler(ds, nb), pol)
    ev.yield_sms = ys
    print(rank, "start", flush=True)
    print(rank, ev(mt.MaternParams(1.0, 0.1, 0.5)), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    for tag, ys in (("dp", 0), ("mp", 0), ("mp", 32)):
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
        ctx = mp.get_context("spawn")
        ps = [ctx.Process(target=worker, args=(r, 2, port, tag, ys)) for r in range(2)]
        for p in ps: p.start()
        for p in ps: p.join(120)
        print(tag, ys, "exit codes", [p.exitcode for p in ps], flush=True)
