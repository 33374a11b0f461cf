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


# ---------------------------------------------------------------- one problem across ranks
def _shard_worker(rank, world, port, out):
    """each rank: the oracle's normal equations of its half of C1 at a pose, all-reduced over
    gloo (the exchange step of the split path), then the same solve on every rank"""
    import numpy as np
    import oracle
    from tests import workloads as W
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = W.c1()
        half = w.m // 2
        sl = slice(0, half) if rank == 0 else slice(half, w.m)
        pose = np.eye(4)
        o = oracle.icp_system(w.target, w.target_normals, w.source[sl], pose, "point_to_plane", w.max_dist, brute=True)
        v = torch.tensor(np.concatenate([o.H.ravel(), o.g, [o.sse, float(o.count)]]), dtype=torch.float64)
        dist.all_reduce(v, op=dist.ReduceOp.SUM)
        H, g, cnt = v[:36].numpy().reshape(6, 6), v[36:42].numpy(), int(v[43].item())
        st, P, *_ = oracle.solve_update(H, g, cnt, pose)
        out[rank] = (st, P.tolist())
    finally:
        dist.destroy_process_group()


def test_split_problem_allreduce_gloo_world2():
    import numpy as np
    import oracle
    from tests import workloads as W
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_shard_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] == out[1]                                 # identical pose on every rank
    w = W.c1()
    o = oracle.icp_system(w.target, w.target_normals, w.source, np.eye(4), "point_to_plane", w.max_dist, brute=True)
    st, P, *_ = oracle.solve_update(o.H, o.g, o.count, np.eye(4))
    assert out[0][0] == st == 0
    np.testing.assert_allclose(np.array(out[0][1]), P, rtol=0, atol=1e-12)   # linearity of the split


def _driver_worker(rank, world, port, out):
    """icp_run_distributed's control flow with the shard steps stubbed by the oracle (no GPU):
    one SUM all-reduce of the 32 sums per iteration, the same pose on every rank.  The package
    is imported as is (loading libcil.so needs no GPU) and its ShardRun is replaced by a stub
    that computes the shard's normal equations with the oracle."""
    import numpy as np
    import oracle
    import paper_1807_00399_b200 as cil
    from tests import workloads as W
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = W.c1()
        half = w.m // 2
        sl = slice(0, half) if rank == 0 else slice(half, w.m)

        class FakeRun:
            def __init__(self, t, src_shard, pose_init, params, stream=None):
                self.P = np.eye(4)
                self.iter_log = []

            def accumulate(self):
                o = oracle.icp_system(w.target, w.target_normals, w.source[sl], self.P, "point_to_plane",
                                      w.max_dist, brute=True)
                self.sums = torch.zeros(44, dtype=torch.float64)
                self.sums[:36] = torch.tensor(o.H.ravel()); self.sums[36:42] = torch.tensor(o.g)
                self.sums[42] = o.sse; self.sums[43] = float(o.count)
                return self.sums

            def finish(self):
                v = self.sums.numpy()
                st, self.P, *_ = oracle.solve_update(v[:36].reshape(6, 6), v[36:42], int(v[43]), self.P)

            def result(self):
                return self.P

        cil.ShardRun = FakeRun

        class Prm:
            max_iters = 3
        P, _ = cil.icp_run_distributed(None, None, None, Prm)
        out[rank] = P.tolist()
    finally:
        dist.destroy_process_group()


def test_icp_run_distributed_driver_gloo_world2():
    import numpy as np
    import oracle
    from tests import workloads as W
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_driver_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] == out[1]
    w = W.c1()
    r = oracle.icp_run(w.target, w.target_normals, w.source, "point_to_plane", 3, w.max_dist, brute=True)
    np.testing.assert_allclose(np.array(out[0]), r.pose, rtol=0, atol=1e-10)
