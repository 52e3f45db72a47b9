"""The N > 1 path of bench.py on CPU: world_size-2 gloo ranks shard the output batch
(longest-first round robin by exact path count) with no data-path collective; the only
collectives are the timing max and the path/output sums, as in bench.py."""
import os
import socket

import numpy as np
import pytest
import torch
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
    mine = bench.shard(P, rank, world)
    local_ms = float(10 + rank)  # stand-in for the rank's device time
    t = torch.tensor([local_ms], dtype=torch.float64)
    tot = torch.tensor([float(P[mine].astype(np.float64).sum()), float(len(mine))], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    out[rank] = (mine.tolist(), float(t.item()), tot.tolist())
    dist.destroy_process_group()


def test_two_rank_sharding_and_reductions():
    import bench
    d = np.load(os.path.join(os.path.dirname(bench.__file__), "data", "cfg4.npz"))
    P = d["P_cond"][:4001]  # odd size: ranks get different counts
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), P, out), nprocs=world, join=True)
    shards = [out[r][0] for r in range(world)]
    allidx = sorted(shards[0] + shards[1])
    assert allidx == list(range(len(P)))  # every output exactly once
    assert not set(shards[0]) & set(shards[1])
    for r in range(world):
        assert out[r][1] == 11.0  # max over ranks of the device time
        assert out[r][2][0] == pytest.approx(float(P.astype(np.float64).sum()))
        assert out[r][2][1] == len(P)
    w = [float(P[s].astype(np.float64).sum()) for s in shards]
    assert abs(w[0] - w[1]) / sum(w) < 0.01  # longest-first round robin balances path counts
