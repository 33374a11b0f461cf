"""CPU (gloo, world_size 2) checks of bench.py's multi-GPU path: whole-job aggregation is the
max over ranks of the device-timed region and the sum of every rank's point-pairs; every rank
aligns its own seeded frame pair (weak scaling, no data-path collective); the reference arm
runs on rank 0 only."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tot_ms = [12.5, 17.25][rank]
        pairs = [1000.0, 3000.0][rank]
        t, p = bench.reduce_over_ranks(tot_ms, pairs, world, torch.device("cpu"))
        out[rank] = (t, p, bench.rank_seed(rank))
    finally:
        dist.destroy_process_group()


def test_reduce_over_ranks_gloo_world2():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for r in (0, 1):
        t, p, seed = out[r]
        assert t == 17.25                 # max over ranks
        assert p == 4000.0                # sum over ranks
    assert out[0][2] != out[1][2]         # independent frame pairs per rank


def test_single_rank_is_identity():
    assert bench.reduce_over_ranks(3.0, 7.0, 1, None) == (3.0, 7.0)


def test_reference_arm_runs_on_rank0_only():
    class A:
        workload = "c1"; iters = 0; warmup = 0; steps = 1; cpu_sample = 256
    assert bench.run_reference(A, 1, 2) is None


def test_rank_workloads_differ():
    import gen
    a = gen.c1_sphere(base=bench.rank_seed(0))
    b = gen.c1_sphere(base=bench.rank_seed(1))
    assert a.target.shape == b.target.shape
    assert not (a.target == b.target).all()
