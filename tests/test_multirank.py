"""N > 1 host logic on CPU with the gloo backend (world_size 2): the bench shards the
independent systems of a sequence across ranks (weak scaling, no data-path
collective) and aggregates max-over-ranks time and summed solves."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids = bench.systems_for_rank(rank, 5, 20)
    # each rank solves its own tiny systems with the oracle (stand-in for the GPU step) and times it
    import oracle as orc
    import synth
    its = []
    for s in ids[:2]:
        sy = synth.system(1, s, n=12)
        A = orc.Csr(sy.rp, sy.ci, sy.val)
        x, it, st, _ = orc.pcg(A, sy.b, sy.x0)
        assert st == 0
        its.append(it)
    ms = 100.0 + 50.0 * rank
    ms_max, value = bench.aggregate(ms, 3 * len(ids), world, dist, None)
    gathered = [None] * world
    dist.all_gather_object(gathered, ids)
    if rank == 0:
        out.put((ms_max, value, gathered))
    dist.destroy_process_group()


def test_two_rank_sharding_and_aggregation():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    ms_max, value, gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ms_max == 150.0                              # max over ranks
    assert value == pytest.approx(2 * 15 / 0.150)       # summed solves / max time
    assert set(gathered[0]).isdisjoint(gathered[1])     # independent problems per rank
    assert all(0 <= s < 20 for g in gathered for s in g)


def test_single_rank_aggregate_is_identity():
    ms, v = bench.aggregate(200.0, 6, 1)
    assert ms == 200.0 and v == pytest.approx(30.0)
