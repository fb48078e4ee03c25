"""world_size-2 gloo tests (CPU) of the multi-GPU host logic: shard ranges,
max-over-ranks timing, and the SUM assembly used by the verification gather."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_2504_16922_b200.shard import balanced_range, unit_range, work_range

        res = {}
        # every unit / work item owned by exactly one rank
        for total in (0, 1, 7, 24, 10896, 10897):
            b, e = work_range(total, world, rank)
            got = [None] * world
            dist.all_gather_object(got, (b, e))
            cover = sorted(x for (b2, e2) in got for x in range(b2, e2))
            res[("cover", total)] = cover == list(range(total))
            res[("balance", total)] = max(e2 - b2 for b2, e2 in got) - min(e2 - b2 for b2, e2 in got) <= 1
        ub, ue = unit_range(1, 24, world, rank)
        res["units"] = (ub, ue)
        # max over ranks of device times (bench helper)
        m = bench._max_over_ranks([float(rank + 1), 10.0 - rank], world, torch.device("cpu"))
        res["max"] = m
        # verification assembly: disjoint shards over zeros, SUM == full
        full = torch.arange(100, dtype=torch.float32) * 0.5 - 7
        b, e = balanced_range(100, world, rank)
        shard = torch.zeros(100)
        shard[b:e] = full[b:e]
        dist.all_reduce(shard, op=dist.ReduceOp.SUM)
        res["assembled"] = bool(torch.equal(shard, full))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_two_rank_gloo_host_logic():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=150) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, res in results.items():
        for key, val in res.items():
            if key[0] in ("cover", "balance"):
                assert val, (rank, key)
        assert res["max"] == [2.0, 10.0]
        assert res["assembled"]
    assert results[0]["units"] == (0, 12) and results[1]["units"] == (12, 24)
