"""GPU parity at BASELINE.json's full sizes, in the configuration bench.py times (C4: the 2 M-point
LiDAR frame pair, point-to-plane, 50 iterations, certified warm start), and C5 at 2^22 and 2^24
points -- against the fp64 oracle: every query where the oracle can afford it (C4 iterate, C5
2^22), a seeded sample of the queries otherwise (C5 2^24), and the final pose of the 50-iteration
run against the oracle's own 50-iteration run.  Tolerances as tests/test_gpu_parity.py."""
import numpy as np
import pytest
import torch

import oracle
from tests import workloads as W
from tests.test_gpu_parity import _perturb, check_iteration, check_nn, dev

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def cil():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1807_00399_b200 as cil
    return cil


@pytest.mark.parametrize("frac", [0.0, 1.0])
def test_iterate_c4_full(cil, frac):
    """one stateless iteration on the full C4 frame pair: every correspondence, H, g, pose"""
    w = W.c4("point_to_plane")
    check_iteration(cil, w, _perturb(w.gt_pose, frac), "point_to_plane")


@pytest.mark.parametrize("metric", ["point_to_plane", "point_to_point"])
def test_run_c4_full_bench_configuration(cil, metric):
    """the bench's run (50 iterations, certified warm start) against the oracle's 50 full
    iterations, and bit for bit against 50 chained stateless GPU iterations -- for both C4
    variants (BASELINE.json configs[3] "point-to-point and point-to-plane variants"; the
    point-to-point run has the slowest certificate dynamics)"""
    w = W.c4(metric)
    nrm = dev(w.target_normals) if metric == "point_to_plane" else None
    t = cil.cil_target_build(dev(w.target), nrm)
    prm = cil.make_params(metric, w.max_iters, w.max_dist)
    res_t, log = cil.cil_icp_run(t, dev(w.source), dev(np.eye(4)), prm)
    res = cil.decode_result(res_t)
    o = oracle.icp_run(None, w.target_normals if metric == "point_to_plane" else None, w.source, metric,
                       w.max_iters, w.max_dist, tree=W.oracle_tree(w))
    assert res.status == o.status == 0 and res.iterations == o.iterations == w.max_iters
    dr = W.rot_angle(res.pose[:3, :3] @ o.pose[:3, :3].T)
    dt = np.abs(res.pose[:3, 3] - o.pose[:3, 3]).max()
    assert dr <= 1e-4 and dt <= 1e-5, (dr, dt)
    np.testing.assert_allclose(log.cpu().numpy()[:, 0], o.iter_log[:, 0], rtol=1e-4, atol=3)
    P = dev(np.eye(4))
    src = dev(w.source)
    for _ in range(w.max_iters):
        P, *_ = cil.cil_icp_iterate(t, src, P, prm, want_sys=False)
    assert np.array_equal(P.cpu().numpy(), res.pose)


@pytest.mark.parametrize("frac", [0.0, 1.0])
def test_iterate_c4_point_to_point_full(cil, frac):
    w = W.c4("point_to_point")
    check_iteration(cil, w, _perturb(w.gt_pose, frac), "point_to_point")


def test_iterate_c5_2e22_every_query(cil):
    w = W.c5(22)
    check_iteration(cil, w, np.eye(4), "point_to_plane")


def test_iterate_c5_2e24_sampled(cil):
    """2^24 points: GPU correspondences on a seeded 200k-query sample checked one by one
    against the oracle's exact 2-NN; H and g through the GPU's own correspondences (R17)"""
    w = W.c5(24)
    t = cil.cil_target_build(dev(w.target), dev(w.target_normals))
    prm = cil.make_params("point_to_plane", 1, w.max_dist)
    pose_out, sys_t, ci, cd = cil.cil_icp_iterate(t, dev(w.source), dev(np.eye(4)), prm, want_corr=True)
    gs = cil.decode_system(sys_t)
    g_idx = ci.cpu().numpy()
    g_d2 = cd.cpu().numpy()
    rng = np.random.default_rng(24)
    smp = np.sort(rng.choice(w.m, 200_000, replace=False))
    q = w.source[smp].astype(np.float64)
    o_idx, o_d2 = oracle.knn(None, q, k=2, max_dist=w.max_dist, tree=W.oracle_tree(w))
    check_nn(w.target, q, g_idx[smp], g_d2[smp], o_idx, o_d2, max_d2=w.max_dist ** 2)
    assert gs.status == cil.CIL_OK
    r = oracle.icp_system_from_corr(w.target, w.target_normals, w.source, np.eye(4), "point_to_plane",
                                    g_idx.astype(np.int32))
    assert r.count == gs.n_corr
    relH = np.linalg.norm(gs.H - r.H) / np.linalg.norm(r.H)
    relg = np.linalg.norm(gs.g - r.g) / max(np.linalg.norm(r.g), 1e-3 * np.linalg.norm(r.gabs))
    assert relH <= 1e-6 and relg <= 1e-5, (relH, relg)
