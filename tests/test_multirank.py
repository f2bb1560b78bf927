"""Multi-rank harness logic on CPU (gloo, world size 2): replicas, max-over-ranks timing,
whole-job throughput.  The solve itself does not shard (DESIGN.md "Multi-GPU: replicas
only"), so there is no data-path collective to test."""
import os
import socket

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
    t = 10.0 + 5.0 * rank                      # rank 1 is the slow replica
    tmax = bench.aggregate_time(t, dist)
    out[rank] = (tmax, bench.job_throughput(world, 4, tmax))
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_and_throughput():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0][0] == out[1][0] == 15.0
    assert out[0][1] == pytest.approx(2 * 4 / 0.015)


def test_single_rank_passthrough():
    assert bench.aggregate_time(12.5, None) == 12.5
    assert bench.job_throughput(1, 10, 1000.0) == pytest.approx(10.0)
