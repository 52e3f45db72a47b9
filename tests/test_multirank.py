"""The N > 1 path of bench.py on CPU: world_size-2 gloo ranks each evaluate the whole
batch (weak scaling: outputs are independent, so there is no data-path collective); the
only collectives are the timing max and the path/output sums, as in bench.py."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, P, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    local_ms = float(10 + rank)  # stand-in for the rank's device time
    res = bench.aggregate(local_ms, float(P.astype(np.float64).sum()), float(len(P)), world, dist, None)
    out[rank] = res
    dist.destroy_process_group()


def test_two_rank_weak_scaling_reductions():
    import bench
    d = np.load(os.path.join(os.path.dirname(bench.__file__), "data", "cfg4.npz"))
    P = d["P_cond"][:4001]
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), P, out), nprocs=world, join=True)
    for r in range(world):
        t, paths, outs = out[r]
        assert t == 11.0  # max over ranks of the device time
        assert paths == world * float(P.astype(np.float64).sum())  # whole-job paths
        assert outs == world * len(P)
