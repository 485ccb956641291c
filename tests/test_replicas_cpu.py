"""The N>1 benchmark path on CPU: two gloo ranks run independent replicas and
combine timings as the bench does (max over ranks, total solves / max time).
No data-path collective exists (replicas only)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist

    import bench

    dist.init_process_group("gloo", rank=rank, world_size=world)
    ms_local = 100.0 * (rank + 1)  # the slower replica sets the job time
    value, ms_max = bench.replica_value(dist, world, steps=3, ms_local=ms_local)
    bench.barrier(dist)
    q.put((rank, value, ms_max))
    dist.destroy_process_group()


def test_two_rank_replicas_take_max_over_ranks():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, value, ms_max in out:
        assert ms_max == pytest.approx(200.0)
        assert value == pytest.approx(world * 3 / 0.2)
