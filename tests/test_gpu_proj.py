"""GPU parity of the projective data-association engine (cil_proj_iterate / cil_proj_run;
SURVEY.md 8(f) NEXT-2, R23-R26) against the fp64 oracle (oracle.proj_system /
proj_run) on the same seeded inputs, through the C ABI.

Correspondences are pixel indices: bit-exact except inside the rounding band (the unrounded
u or v within 1e-6 px of a half-integer, R24) and the rejection band (R2); H within 1e-5
relative Frobenius and g within 1e-5 of ||g|| (R16), and to 1e-6 after reconciling through
the GPU's own correspondences (R17); poses within 1e-4 rad / 1e-5 units.
"""
import math

import numpy as np
import pytest
import torch
from scipy.spatial.transform import Rotation

import gen
import oracle
from tests import workloads as W

pytestmark = pytest.mark.gpu

ROUND_BAND = 1e-6
BAND = 2e-6
C3_INTR = (640, 480, gen.FX, gen.FY, gen.CX, gen.CY)
COMBINED_W = (0.4, 1.3)


@pytest.fixture(scope="module")
def cil():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1807_00399_b200 as cil
    return cil


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a)).cuda()


def _pose(R=np.eye(3), t=np.zeros(3)):
    T = np.eye(4)
    T[:3, :3] = R
    T[:3, 3] = t
    return T


def _perturb(gt, frac):
    rv = Rotation.from_matrix(gt[:3, :3]).as_rotvec() * frac
    return _pose(Rotation.from_rotvec(rv).as_matrix(), gt[:3, 3] * frac)


def _params(cil, metric, iters, max_dist):
    if metric == "combined":
        oracle.set_combined_weights(*COMBINED_W)
        return cil.make_params(metric, iters, max_dist, w_point=COMBINED_W[0], w_plane=COMBINED_W[1])
    return cil.make_params(metric, iters, max_dist)


def check_proj_iteration(cil, tgt, nrm, intr, src, pose, metric, max_dist):
    K = cil.make_intrinsics(*intr)
    prm = _params(cil, metric, 1, max_dist)
    pose_out, sys_t, ci, cd = cil.cil_proj_iterate(dev(tgt), dev(nrm) if nrm is not None else None, K, dev(src),
                                                   dev(pose.astype(np.float64)), prm, want_corr=True)
    gs = cil.decode_system(sys_t)
    g_idx = ci.cpu().numpy().astype(np.int64)
    g_d2 = cd.cpu().numpy().astype(np.float64)
    o = oracle.proj_system(tgt, nrm, intr, src, pose, metric, max_dist)
    # correspondences: bit-exact outside the bands
    diff = g_idx != o.corr_idx
    if diff.any():
        uv = o.uv[diff]
        fr = np.abs(uv - np.floor(uv) - 0.5)
        in_round = (fr < ROUND_BAND * np.maximum(1.0, np.abs(uv))).any(1)
        s64 = oracle.transform(pose, src[diff])
        in_rej = np.zeros(diff.sum(), bool)
        for cand in (g_idx[diff], o.corr_idx[diff]):
            ok = cand >= 0
            d2 = ((s64[ok] - tgt[cand[ok]].astype(np.float64)) ** 2).sum(1)
            in_rej[np.flatnonzero(ok)] |= np.abs(d2 / max_dist ** 2 - 1.0) <= BAND
        bad = ~(in_round | in_rej)
        assert not bad.any(), f"{bad.sum()} of {diff.sum()} pixel correspondences differ outside the bands"
    both = (g_idx >= 0) & (g_idx == o.corr_idx)
    err = np.abs(g_d2[both] - o.corr_d2[both])
    assert (err <= 1e-6 * o.corr_d2[both] + 1e-30).all(), np.max(err / np.maximum(o.corr_d2[both], 1e-300))
    assert np.all(np.isinf(g_d2[g_idx < 0]))
    if o.count == 0:
        assert gs.n_corr == 0 and gs.status == cil.CIL_NO_CORRESPONDENCES
        assert np.array_equal(pose_out.cpu().numpy(), pose)
        return gs, g_idx, o
    assert gs.status == o_status(o) and abs(gs.n_corr - o.count) <= max(2, 1e-5 * o.count)
    relH = np.linalg.norm(gs.H - o.H) / np.linalg.norm(o.H)
    gscale = max(np.linalg.norm(o.g), 1e-3 * np.linalg.norm(o.gabs))
    relg = np.linalg.norm(gs.g - o.g) / gscale
    assert relH <= 1e-5 and relg <= 1e-5, (relH, relg)
    r = oracle.icp_system_from_corr(tgt, nrm, src, pose, metric, g_idx.astype(np.int32))
    assert r.count == gs.n_corr
    relH2 = np.linalg.norm(gs.H - r.H) / np.linalg.norm(r.H)
    relg2 = np.linalg.norm(gs.g - r.g) / max(np.linalg.norm(r.g), 1e-3 * np.linalg.norm(r.gabs))
    assert relH2 <= 1e-6 and relg2 <= 1e-5, (relH2, relg2)
    if gs.status == cil.CIL_OK:
        st, Pr, *_ = oracle.solve_update(gs.H, gs.g, gs.n_corr, pose)
        Pg = pose_out.cpu().numpy()
        assert W.rot_angle(Pg[:3, :3] @ Pr[:3, :3].T) < 1e-12 and np.abs(Pg[:3, 3] - Pr[:3, 3]).max() < 1e-12
        st, Po, *_ = oracle.solve_update(o.H, o.g, o.count, pose)
        assert W.rot_angle(Pg[:3, :3] @ Po[:3, :3].T) < 1e-4 and np.abs(Pg[:3, 3] - Po[:3, 3]).max() < 1e-5
    return gs, g_idx, o


def o_status(o):
    st, *_ = oracle.solve_update(o.H, o.g, o.count, np.eye(4))
    return st


@pytest.mark.parametrize("metric", ["point_to_plane", "point_to_point", "combined"])
@pytest.mark.parametrize("frac", [0.0, 0.5, 1.0])
def test_proj_iterate_c3(cil, metric, frac):
    w = W.c3()
    check_proj_iteration(cil, w.target, w.target_normals, C3_INTR, w.source, _perturb(w.gt_pose, frac), metric,
                         w.max_dist)


def test_proj_iterate_invalid_pixels(cil):
    """invalid target pixels (z <= 0, z < 0, NaN) never pair (R23)"""
    w = W.c3()
    tgt = w.target.copy()
    rng = np.random.default_rng(7)
    tgt[rng.random(tgt.shape[0]) < 0.1, 2] = 0.0
    tgt[50000:60000, 2] = -1.0
    tgt[rng.integers(0, tgt.shape[0], 500)] = np.nan
    gs, g_idx, o = check_proj_iteration(cil, tgt, w.target_normals, C3_INTR, w.source, _perturb(w.gt_pose, 0.5),
                                        "point_to_plane", w.max_dist)
    ok = g_idx >= 0
    assert np.all(tgt[g_idx[ok], 2] > 0) and np.all(np.isfinite(tgt[g_idx[ok]]))


@pytest.mark.parametrize("w_img,h_img,m", [(1, 1, 1), (37, 23, 851), (64, 48, 3072), (101, 7, 100003)])
def test_proj_iterate_small_ragged(cil, w_img, h_img, m):
    """odd image shapes and source sizes that are not multiples of the CTA tile"""
    rng = np.random.default_rng(w_img * 1000 + m)
    fx, fy = 0.8 * w_img + 1.0, 0.8 * w_img + 1.0
    cx, cy = (w_img - 1) / 2.0, (h_img - 1) / 2.0
    u, v = np.meshgrid(np.arange(w_img, dtype=np.float64), np.arange(h_img, dtype=np.float64))
    z = 2.0 + 0.3 * np.sin(u / 5.0) + 0.2 * np.cos(v / 3.0)
    tgt = np.stack([(u - cx) * z / fx, (v - cy) * z / fy, z], -1).reshape(-1, 3).astype(np.float32)
    nrm = rng.standard_normal(tgt.shape)
    nrm = (nrm / np.linalg.norm(nrm, axis=1, keepdims=True)).astype(np.float32)
    src = (tgt[rng.integers(0, tgt.shape[0], m)] + rng.normal(0, 0.02, (m, 3))).astype(np.float32)
    pose = _pose(Rotation.from_rotvec([0.01, -0.02, 0.015]).as_matrix(), np.array([0.02, -0.01, 0.03]))
    for metric in ("point_to_plane", "point_to_point"):
        check_proj_iteration(cil, tgt, nrm, (w_img, h_img, fx, fy, cx, cy), src, pose, metric, 0.2)


def test_proj_rounding_half_away_from_zero(cil):
    """exact half-pixel projections (fx = 1, z = 1: u = x exactly) round away from zero on the
    GPU too, then the bounds check (R24) -- the oracle pin's case, bit-exact"""
    intr = (4, 1, 1.0, 1.0, 0.0, 0.0)
    src = np.array([[0.5, 0.0, 1.0], [2.5, 0.0, 1.0], [-0.5, 0.0, 1.0], [3.5, 0.0, 1.0],
                    [1.4999999, 0.0, 1.0], [0.0, 0.5, 1.0], [0.0, -0.4, 1.0]], np.float32)
    tgt = np.array([[0.0, 0.0, 1.0], [0.5, 0.0, 1.0], [1.5, 0.0, 1.0], [2.5, 0.0, 1.0]], np.float32)
    K = cil.make_intrinsics(*intr)
    _, _, ci, cd = cil.cil_proj_iterate(dev(tgt), None, K, dev(src), dev(np.eye(4)),
                                        cil.make_params("point_to_point", 1, 10.0), want_corr=True)
    np.testing.assert_array_equal(ci.cpu().numpy(), [1, 3, -1, -1, 1, -1, 0])


def test_proj_no_correspondences_and_empty(cil):
    """everything behind the camera -> CIL_NO_CORRESPONDENCES, pose unchanged; m = 0 likewise"""
    w = W.c3()
    K = cil.make_intrinsics(*C3_INTR)
    flip = _pose(Rotation.from_rotvec([math.pi, 0.0, 0.0]).as_matrix())
    P = dev(flip)
    out, sys_t, ci, _ = cil.cil_proj_iterate(dev(w.target), dev(w.target_normals), K, dev(w.source), P,
                                             cil.make_params("point_to_plane", 1, 0.05), want_corr=True)
    gs = cil.decode_system(sys_t)
    assert gs.status == cil.CIL_NO_CORRESPONDENCES and gs.n_corr == 0
    assert np.array_equal(out.cpu().numpy(), flip) and (ci.cpu().numpy() == -1).all()
    empty = torch.empty((0, 3), dtype=torch.float32, device="cuda")
    out, sys_t, _, _ = cil.cil_proj_iterate(dev(w.target), dev(w.target_normals), K, empty, dev(np.eye(4)),
                                            cil.make_params("point_to_plane", 1, 0.05))
    assert cil.decode_system(sys_t).status == cil.CIL_NO_CORRESPONDENCES


def check_proj_run(cil, tgt, nrm, intr, src, metric, iters, max_dist, pose_init):
    K = cil.make_intrinsics(*intr)
    prm = _params(cil, metric, iters, max_dist)
    res_t, log = cil.cil_proj_run(dev(tgt), dev(nrm), K, dev(src), dev(pose_init), prm)
    res = cil.decode_result(res_t)
    o = oracle.proj_run(tgt, nrm, intr, src, metric, iters, max_dist, pose_init=pose_init)
    assert res.status == o.status == cil.CIL_OK and res.iterations == o.iterations == iters
    dr = W.rot_angle(res.pose[:3, :3] @ o.pose[:3, :3].T)
    dt = np.abs(res.pose[:3, 3] - o.pose[:3, 3]).max()
    assert dr <= 1e-4 and dt <= 1e-5, (dr, dt)
    lg = log.cpu().numpy()
    np.testing.assert_allclose(lg[:, 0], o.iter_log[:, 0], rtol=1e-4, atol=3)
    np.testing.assert_allclose(lg[:, 1], o.iter_log[:, 1], rtol=1e-3)
    # the device loop equals the chain of stateless iterations bit for bit
    P = dev(pose_init)
    for _ in range(iters):
        P, *_ = cil.cil_proj_iterate(dev(tgt), dev(nrm), K, dev(src), P, prm, want_sys=False)
    assert np.array_equal(P.cpu().numpy(), res.pose)
    return res, o


@pytest.mark.parametrize("metric", ["point_to_plane", "point_to_point", "combined"])
def test_proj_run_c3(cil, metric):
    w = W.c3()
    check_proj_run(cil, w.target, w.target_normals, C3_INTR, w.source, metric, w.max_iters, w.max_dist, np.eye(4))


def test_proj_run_c3_from_ground_truth_and_deterministic(cil):
    w = W.c3()
    res, _ = check_proj_run(cil, w.target, w.target_normals, C3_INTR, w.source, "point_to_plane", 10, w.max_dist,
                            w.gt_pose)
    E = res.pose @ np.linalg.inv(w.gt_pose)
    assert math.degrees(W.rot_angle(E[:3, :3])) < 0.05 and np.linalg.norm(E[:3, 3]) < 2e-3
    K = cil.make_intrinsics(*C3_INTR)
    prm = cil.make_params("point_to_plane", 30, w.max_dist)
    a = [cil.decode_result(cil.cil_proj_run(dev(w.target), dev(w.target_normals), K, dev(w.source), dev(np.eye(4)),
                                            prm)[0]).pose for _ in range(2)]
    assert np.array_equal(a[0], a[1])


def test_proj_run_empty_source_and_convergence_stop(cil):
    """the persistent loop with an empty source stops at iteration 1 with CIL_NO_CORRESPONDENCES;
    with convergence tolerances it stops at the oracle's iteration with the oracle's pose"""
    w = W.c3()
    K = cil.make_intrinsics(*C3_INTR)
    empty = torch.empty((0, 3), dtype=torch.float32, device="cuda")
    res = cil.decode_result(cil.cil_proj_run(dev(w.target), dev(w.target_normals), K, empty, dev(np.eye(4)),
                                             cil.make_params("point_to_plane", 5, 0.05))[0])
    assert res.status == cil.CIL_NO_CORRESPONDENCES and res.iterations == 1 and np.array_equal(res.pose, np.eye(4))
    prm = cil.make_params("point_to_plane", 300, 0.05, rot_tol=1e-5, trans_tol=1e-5)
    res = cil.decode_result(cil.cil_proj_run(dev(w.target), dev(w.target_normals), K, dev(w.source), dev(np.eye(4)),
                                             prm)[0])
    o = oracle.proj_run(w.target, w.target_normals, C3_INTR, w.source, "point_to_plane", 300, 0.05,
                        rot_tol=1e-5, trans_tol=1e-5)
    assert res.converged and o.converged and abs(res.iterations - o.iterations) <= 1
    assert W.rot_angle(res.pose[:3, :3] @ o.pose[:3, :3].T) <= 1e-4 and np.abs(res.pose[:3, 3] - o.pose[:3, 3]).max() <= 1e-5
