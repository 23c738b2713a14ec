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


def _sweep_worker(rank, world, port, cfg_path, out):
    """cli sweep under 2 gloo ranks with the GPU solve replaced by a stub:
    points are sharded round-robin, rank 0 prints every row in point order."""
    import contextlib
    import io as _io
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1907_13428_b200 import cli
    from paper_1907_13428_b200 import io as fio

    def fake_point(p, ctx=None):
        # every point of a rank is solved on that rank's own device context
        assert ctx == ("ctx", rank), ctx
        res = {"status": "converged" if p.admm.delta < 1.0 else "itercap", "iterations": int(10 * p.admm.delta),
               "pcg_avg": float(rank), "misfit": 0.5, "dual_inf": 1e-9, "wall_seconds": 0.0}
        return fio.make_summary_row(p, p.admm.delta, res), (0 if res["status"] == "converged" else 2)
    cli._run_point = fake_point
    cli._rank_context = lambda local: ("ctx", local)
    buf = _io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.main(["sweep", "--config", cfg_path])
    out[rank] = (rc, buf.getvalue())
    dist.destroy_process_group()


def test_cli_sweep_sharded_gloo(tmp_path):
    cfg = tmp_path / "s.cfg"
    cfg.write_text("n = 4\ndelta_sweep = 0.2, 0.4, 0.8, 1.2, 1.5\n")
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_sweep_worker, args=(2, _free_port(), str(cfg), out), nprocs=2, join=True)
    rc0, txt0 = out[0]
    rc1, txt1 = out[1]
    assert rc1 == 0 and txt1 == ""
    lines = txt0.strip().splitlines()
    assert rc0 == 2 and lines[0].startswith("n,N,alpha")
    rows = [ln.split(",") for ln in lines[1:]]
    assert [r[6] for r in rows] == ["0.2", "0.4", "0.8", "1.2", "1.5"]
    assert [r[10] for r in rows] == ["0", "1", "0", "1", "0"]  # pcg_avg = the rank that ran the point
    assert [r[13] for r in rows] == ["converged"] * 3 + ["itercap"] * 2
