"""GPU parity of the multi-GPU split of one ICP problem (cil_icp_shard_*),
exercised on one GPU with the ranks' shards run one after another and their 32 fp64 sums added
on the device in rank order (exactly what an all-reduce delivers): every shard ends with the
bitwise same pose, equal to the unsplit cil_icp_run up to the reduction order (1e-9) and to the
oracle within the north_star tolerance (1e-4 rad, 1e-5)."""
import numpy as np
import pytest
import torch

import oracle
from tests import workloads as W

pytestmark = pytest.mark.gpu

COMBINED_W = (0.4, 1.3)


@pytest.fixture(scope="module")
def cil():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1807_00399_b200 as cil
    return cil


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a)).cuda()


def _params(cil, metric, iters, max_dist):
    if metric == "combined":
        oracle.set_combined_weights(*COMBINED_W)
        return cil.make_params(metric, iters, max_dist, w_point=COMBINED_W[0], w_plane=COMBINED_W[1])
    return cil.make_params(metric, iters, max_dist)


@pytest.mark.parametrize("metric", ["point_to_plane", "point_to_point", "combined"])
def test_shards_equal_unsplit_run(cil, metric):
    w = W.c4("point_to_plane" if metric == "combined" else metric, rings=16, az=8000)
    t = cil.cil_target_build(dev(w.target), dev(w.target_normals))
    prm = _params(cil, metric, w.max_iters, w.max_dist)
    m = w.m
    cuts = [0, int(0.4 * m), int(0.4 * m), int(0.75 * m), m]          # 4 ranks, one empty shard
    shards = [cil.ShardRun(t, dev(w.source[a:b]), dev(np.eye(4)), prm) for a, b in zip(cuts[:-1], cuts[1:])]
    for _ in range(w.max_iters):
        tot = torch.zeros(32, dtype=torch.float64, device="cuda")
        for r in shards:
            tot += r.accumulate()
        for r in shards:
            r.finish(tot)
    res = [cil.decode_result(r.result()) for r in shards]
    for r in res[1:]:
        assert np.array_equal(r.pose, res[0].pose) and r.n_corr == res[0].n_corr and r.iterations == res[0].iterations
    logs = [r.iter_log.cpu().numpy() for r in shards]
    for lg in logs[1:]:
        assert np.array_equal(lg, logs[0])
    full, flog = cil.cil_icp_run(t, dev(w.source), dev(np.eye(4)), prm)
    fr = cil.decode_result(full)
    assert res[0].status == fr.status == cil.CIL_OK and res[0].iterations == fr.iterations
    assert W.rot_angle(res[0].pose[:3, :3] @ fr.pose[:3, :3].T) <= 1e-9
    assert np.abs(res[0].pose[:3, 3] - fr.pose[:3, 3]).max() <= 1e-9
    np.testing.assert_allclose(logs[0][:, 0], flog.cpu().numpy()[:, 0], atol=2)
    o = oracle.icp_run(None, w.target_normals, w.source, metric, w.max_iters, w.max_dist, tree=W.oracle_tree(w))
    assert W.rot_angle(res[0].pose[:3, :3] @ o.pose[:3, :3].T) <= 1e-4
    assert np.abs(res[0].pose[:3, 3] - o.pose[:3, 3]).max() <= 1e-5


def test_shard_stop_rules(cil):
    """convergence tolerances stop every shard at the same iteration (the stop flag comes from
    the shared solve)"""
    w = W.c4("point_to_plane", rings=16, az=8000)
    t = cil.cil_target_build(dev(w.target), dev(w.target_normals))
    prm = cil.make_params("point_to_plane", 50, w.max_dist, rot_tol=1e-4, trans_tol=1e-4)   # oracle: stops at 17
    half = w.m // 2
    shards = [cil.ShardRun(t, dev(w.source[:half]), dev(np.eye(4)), prm),
              cil.ShardRun(t, dev(w.source[half:]), dev(np.eye(4)), prm)]
    for _ in range(prm.max_iters):
        tot = shards[0].accumulate() + shards[1].accumulate()
        for r in shards:
            r.finish(tot)
    a, b = (cil.decode_result(r.result()) for r in shards)
    full = cil.decode_result(cil.cil_icp_run(t, dev(w.source), dev(np.eye(4)), prm)[0])
    assert a.converged and b.converged and a.iterations == b.iterations == full.iterations < 50
    assert np.array_equal(a.pose, b.pose)


def test_distributed_driver_on_a_side_stream(cil):
    """icp_run_distributed through a real process group (NCCL, world size 1) with a stream that
    is NOT the current one: the driver makes it current for every step, so the all-reduce is
    ordered after the accumulation that writes the sums; the pose equals the unsplit run's
    (same shard = the whole source, the same reduction order)."""
    import os
    import socket
    import torch.distributed as dist
    w = W.c4("point_to_plane", rings=16, az=8000)
    t = cil.cil_target_build(dev(w.target), dev(w.target_normals))
    src = dev(w.source)
    prm = cil.make_params("point_to_plane", 12, w.max_dist)
    res_t, _ = cil.cil_icp_run(t, src, dev(np.eye(4)), prm)
    ref = cil.decode_result(res_t)
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        side = torch.cuda.Stream()
        P0 = dev(np.eye(4))
        side.wait_stream(torch.cuda.current_stream())
        res_d, _ = cil.icp_run_distributed(t, src, P0, prm, stream=side)
        torch.cuda.synchronize()
        got = cil.decode_result(res_d)
    finally:
        dist.destroy_process_group()
    assert got.status == ref.status == 0 and got.iterations == ref.iterations
    assert np.abs(got.pose - ref.pose).max() <= 1e-9


def test_target_freed_on_another_stream(cil):
    """a target used on a side stream and freed from the default stream: the release waits for
    the side stream's queries (the results stay correct after the free)"""
    rng = np.random.default_rng(3)
    T = rng.random((200_000, 3)).astype(np.float32)
    Q = rng.random((300_000, 3)).astype(np.float32)
    side = torch.cuda.Stream()
    dT, dQ = dev(T), dev(Q)
    side.wait_stream(torch.cuda.current_stream())
    t = cil.cil_target_build(dT, None)
    with torch.cuda.stream(side):
        gi, gd = cil.cil_nn_query(t, dQ)
    t.free()                                   # from the current (default) stream
    junk = torch.empty(64 << 20, dtype=torch.uint8, device="cuda").fill_(7)   # reuse freed memory
    torch.cuda.synchronize()
    from scipy.spatial import cKDTree
    d, i = cKDTree(T.astype(np.float64)).query(Q.astype(np.float64), k=1)
    assert (gi.cpu().numpy() == i).mean() > 0.9999
    del junk
