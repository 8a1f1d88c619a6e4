"""N>1 host logic of bench.py on CPU (gloo, world size 2): replicas with no
data-path collective; the whole-job time is the max over ranks and the rate
counts every rank's solves."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    vals = bench.max_over_ranks([10.0 + rank, 5.0 - rank], world)
    rate = bench.whole_job_rate(3, world, vals[0])
    dist.barrier()
    out[rank] = (vals, rate)
    dist.destroy_process_group()


def test_max_over_ranks_and_whole_job_rate_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for rank in range(world):
        vals, rate = res[rank]
        assert vals == [11.0, 5.0]
        assert rate == pytest.approx(2 * 3 / 11e-3)


def test_single_rank_is_identity():
    import bench
    assert bench.max_over_ranks([1.5, 2.5], 1) == [1.5, 2.5]
    assert bench.whole_job_rate(4, 1, 1000.0) == pytest.approx(4.0)
