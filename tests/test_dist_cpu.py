"""The multi-rank plumbing of the weak-scaling run on CPU: world_size 2, gloo,
127.0.0.1 (paper_1801_08914_b200/dist.py; bench.py uses it under torchrun)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1801_08914_b200 import dist as hdist


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w, r, lr = hdist.world()
    assert (w, r, lr) == (world, rank, rank)
    hdist.barrier()
    # per-rank device times -> the max over ranks; units processed -> the sum
    t_max = hdist.reduce_max([1.5 + rank, 10.0 - rank])
    n_sum = hdist.reduce_sum(1000.0 * (rank + 1))
    sh = hdist.shard(10, world, rank)
    out[rank] = (t_max, n_sum, list(sh), hdist.replica_seed(1002, rank))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_gloo_reductions_and_sharding():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for rank in range(world):
        t_max, n_sum, sh, seed = res[rank]
        assert t_max == [2.5, 10.0]
        assert n_sum == 3000.0
    assert res[0][2] + res[1][2] == list(range(10))  # disjoint, complete shards
    assert res[0][3] != res[1][3]                     # distinct replica inputs


def test_single_process_identity():
    assert hdist.reduce_max(3.0) == 3.0 and hdist.reduce_sum([1.0, 2.0]) == [1.0, 2.0]
    assert list(hdist.shard(7, 3, 0)) == [0, 1, 2] and list(hdist.shard(7, 3, 2)) == [5, 6]
