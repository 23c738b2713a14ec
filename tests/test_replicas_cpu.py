"""Multi-rank host logic on CPU (gloo, world_size 2): the hot path runs as
independent replicas; these are the pieces that cross ranks --
sharding of independent solves and the bench's max-time / sum-work reduce."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1907_13428_b200.replicas import aggregate, gather_records, shard
    points = [0.1, 0.4, 1.0, 2.0, 5.0]
    mine = shard(points, rank, world)
    recs = [dict(delta=d, rank=rank) for d in mine]
    t, u = aggregate(10.0 + rank, 3 + rank, dist)
    allrecs = gather_records(recs, dist)
    out[rank] = (mine, t, u, [r["delta"] for r in allrecs])
    dist.destroy_process_group()


def test_replicas_gloo_two_ranks():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    mine0, t0, u0, all0 = out[0]
    mine1, t1, u1, all1 = out[1]
    assert mine0 == [0.1, 1.0, 5.0] and mine1 == [0.4, 2.0]
    assert t0 == t1 == 11.0 and u0 == u1 == 7.0
    assert sorted(all0) == sorted(all1) == [0.1, 0.4, 1.0, 2.0, 5.0]


def test_shard_single_rank_and_errors():
    from paper_1907_13428_b200.replicas import aggregate, shard
    assert shard([1, 2, 3], 0, 1) == [1, 2, 3]
    assert aggregate(5.0, 2) == (5.0, 2.0)
    with pytest.raises(ValueError):
        shard([1], 2, 2)
