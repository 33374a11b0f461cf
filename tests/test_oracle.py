"""Pins for the fp64 CPU oracle (oracle/oracle.c) against things other than itself:
brute force, scipy/numpy library routines, closed forms, finite differences of the true
residual, invariants and planted motions.  CPU only (-m "not gpu").

Each test names the paper passage / DESIGN.md reading it pins.
"""
import math
import os

import numpy as np
import pytest
from scipy.spatial import cKDTree
from scipy.spatial.distance import cdist
from scipy.spatial.transform import Rotation

import gen
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _read_golden(name):
    vals = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            k, *v = line.split()
            if k == "metric":
                vals[k] = v[0]
            else:
                vals.setdefault(k, []).append([float(x) for x in v])
    return vals


def _pose(R=np.eye(3), t=np.zeros(3)):
    T = np.eye(4)
    T[:3, :3] = R
    T[:3, 3] = t
    return T


def _rot_angle(R):
    return math.acos(max(-1.0, min(1.0, (np.trace(R) - 1) / 2)))


# ----------------------------------------------------------------------------- NN
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_kdtree_equals_brute_force(oracle_lib, seed):
    """PAPER.md:122 KDTree k-NN is exact: kd-tree == linear scan, index and d^2, k=1..4."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 2000))
    T = rng.standard_normal((n, 3)).astype(np.float32)
    Q = rng.standard_normal((700, 3))
    tree = oracle.KDTree(T)
    for k in (1, 2, 4):
        i1, d1 = oracle.knn(None, Q, k=k, tree=tree)
        i2, d2 = oracle.knn(T, Q, k=k, brute=True)
        assert np.array_equal(i1, i2) and np.array_equal(d1, d2)


def test_ties_lowest_index(oracle_lib):
    """DESIGN.md R1: equal distances resolve to the lowest target index.
    Integer grid with duplicated points: every duplicate ties exactly."""
    g = np.stack(np.meshgrid(*[np.arange(6)] * 3, indexing="ij"), -1).reshape(-1, 3).astype(np.float32)
    T = np.concatenate([g, g[::-1], g])          # each grid point appears 3 times
    Q = np.concatenate([g.astype(np.float64), g + 0.5, g + 0.25]).astype(np.float64)
    tree = oracle.KDTree(T, leaf=4)
    i1, d1 = oracle.knn(None, Q, k=1, tree=tree)
    D = cdist(Q, T.astype(np.float64), "sqeuclidean")
    ref = np.argmin(D, axis=1)                  # numpy argmin: first (= lowest) index on ties
    assert np.array_equal(i1[:, 0], ref)
    assert np.array_equal(d1[:, 0], D[np.arange(len(Q)), ref])
    # cube centres (g + 0.5) tie between 8 corners x 3 copies: lowest index wins
    assert (i1[:, 0] < len(g)).all()


def test_matches_scipy_ckdtree(oracle_lib):
    """Exact NN distances equal scipy's cKDTree (independent fp64 kd-tree) on a C2-like cloud."""
    rng = np.random.default_rng(5)
    T = rng.random((20000, 3)).astype(np.float32)
    Q = rng.random((5000, 3)).astype(np.float32).astype(np.float64)
    idx, d2 = oracle.knn(T, Q, k=2)
    dd, ii = cKDTree(T.astype(np.float64)).query(Q, k=2)
    np.testing.assert_allclose(d2, dd ** 2, rtol=1e-12, atol=0)
    gap = dd[:, 1] ** 2 - dd[:, 0] ** 2 > 1e-12
    assert np.array_equal(idx[gap, 0], ii[gap, 0])


def test_self_query_and_bound(oracle_lib):
    """SPEC.md:164 self-query returns itself at 0; SPEC.md:389-391 max_dist below every NN
    distance -> no correspondence."""
    rng = np.random.default_rng(3)
    T = rng.random((3000, 3)).astype(np.float32)
    idx, d2 = oracle.knn(T, T.astype(np.float64), k=1)
    assert np.array_equal(idx[:, 0], np.arange(3000)) and (d2 == 0).all()
    Q = T.astype(np.float64) + 10.0
    idx, d2 = oracle.knn(T, Q, k=1, max_dist=1.0)
    assert (idx == -1).all() and np.isinf(d2).all()
    # inclusive bound (R2): a target exactly at max_dist is accepted
    idx, d2 = oracle.knn(np.zeros((1, 3), np.float32), np.array([[0.5, 0.0, 0.0]]), k=1, max_dist=0.5)
    assert idx[0, 0] == 0


def test_empty_target(oracle_lib):
    idx, d2 = oracle.knn(np.zeros((0, 3), np.float32), np.zeros((4, 3)), k=1, brute=True)
    assert (idx == -1).all()


# ----------------------------------------------------------------------------- H, g
@pytest.mark.parametrize("fname", ["single_pair_point_to_plane.txt", "single_pair_point_to_point.txt"])
def test_golden_single_pair(oracle_lib, fname):
    """Hand-worked single-pair systems (tests/golden/)."""
    gd = _read_golden(fname)
    src = np.array(gd["src"], np.float32)
    tgt = np.array(gd["tgt"], np.float32)
    nrm = np.array(gd["nrm"], np.float32) if "nrm" in gd else None
    sys_ = oracle.icp_system(tgt, nrm, src, np.eye(4), gd["metric"], 10.0, brute=True)
    assert sys_.count == 1
    np.testing.assert_array_equal(sys_.g, np.array(gd["g"][0]))
    assert sys_.sse == gd["sse"][0][0]
    if "J" in gd:
        J = np.array(gd["J"][0])
        np.testing.assert_array_equal(sys_.H, np.outer(J, J))
    else:
        np.testing.assert_array_equal(sys_.H, np.array(gd["H"]))


def _residual_fd_jacobian(s, t, n, metric, h=1e-6, w=(0.0, 0.0)):
    """Central finite differences of the TRUE residual r(x) of the rigidly moved point
    s' = Rot(alpha) s + tau (scipy rotation), i.e. an independent construction of J.
    "combined" stacks the weighted residuals [sqrt(w_pp) (s'-t); sqrt(w_pl) (s'-t).n], whose
    least-squares objective is w_pp |s'-t|^2 + w_pl ((s'-t).n)^2 (R22)."""
    def resid(x):
        sp = Rotation.from_rotvec(x[:3]).apply(s) + x[3:]
        if metric == "combined":
            return np.concatenate([np.sqrt(w[0]) * (sp - t), [np.sqrt(w[1]) * np.dot(sp - t, n)]])
        return np.atleast_1d(np.dot(sp - t, n)) if metric == "point_to_plane" else sp - t
    r0 = resid(np.zeros(6))
    J = np.zeros((r0.size, 6))
    for k in range(6):
        e = np.zeros(6)
        e[k] = h
        J[:, k] = (resid(e) - resid(-e)) / (2 * h)
    return r0, J


@pytest.mark.parametrize("metric", ["point_to_plane", "point_to_point", "combined"])
def test_system_equals_finite_difference_jacobian(oracle_lib, metric):
    """H = sum J^T J, g = sum J^T r with J the derivative of the true residual (PAPER.md:140
    [Besl], [Low]).  A dropped term, wrong sign or transposed operand in the
    oracle's J fails here.  Includes a non-identity pose (J uses the transformed point, R4)."""
    rng = np.random.default_rng(11)
    m = 64
    src = rng.uniform(-3, 3, (m, 3)).astype(np.float32)
    pose = _pose(Rotation.from_rotvec([0.1, -0.2, 0.05]).as_matrix(), np.array([0.3, -0.1, 0.2]))
    s = src.astype(np.float64) @ pose[:3, :3].T + pose[:3, 3]
    tgt = (s + rng.normal(0, 0.05, (m, 3))).astype(np.float32)
    nrm = rng.standard_normal((m, 3))
    nrm = (nrm / np.linalg.norm(nrm, axis=1, keepdims=True)).astype(np.float32)
    # correspondences given explicitly (i <-> i) so that this pins only the accumulation
    w = (0.3, 1.7)
    oracle.set_combined_weights(*w)
    sys_ = oracle.icp_system_from_corr(tgt, nrm, src, pose, metric, np.arange(m, dtype=np.int32))
    Hs = np.zeros((6, 6))
    gs = np.zeros(6)
    for i in range(m):
        r0, J = _residual_fd_jacobian(s[i], tgt[i].astype(np.float64), nrm[i].astype(np.float64), metric, w=w)
        Hs += J.T @ J
        gs += J.T @ r0
    scale = np.abs(Hs).max()
    np.testing.assert_allclose(sys_.H, Hs, rtol=0, atol=1e-7 * scale)
    np.testing.assert_allclose(sys_.g, gs, rtol=0, atol=1e-7 * np.abs(gs).max())
    assert sys_.count == m
    # H symmetric PSD
    np.testing.assert_array_equal(sys_.H, sys_.H.T)
    assert np.linalg.eigvalsh(sys_.H).min() > -1e-9 * scale


def test_corr_system_matches_search_system(oracle_lib):
    """orc_icp_system (search) == orc_icp_system_from_corr on its own correspondences."""
    w = gen.c1_sphere()
    pose = _pose(Rotation.from_rotvec([0.01, 0.02, -0.01]).as_matrix(), np.array([0.01, 0, 0]))
    a = oracle.icp_system(w.target, w.target_normals, w.source, pose, "point_to_plane", 0.1)
    b = oracle.icp_system_from_corr(w.target, w.target_normals, w.source, pose, "point_to_plane",
                                    a.corr_idx.astype(np.int32))
    np.testing.assert_array_equal(a.H, b.H)
    np.testing.assert_array_equal(a.g, b.g)
    assert a.count == b.count == int((a.corr_idx >= 0).sum())


# ----------------------------------------------------------------------------- solve / update
@pytest.mark.parametrize("angle", [0.0, 1e-9, 3e-5, 1e-4, 0.3, 2.5])
def test_rodrigues_matches_scipy(oracle_lib, angle):
    """SPEC.md:413 exponential map of alpha == scipy Rotation.from_rotvec (both branches)."""
    axis = np.array([0.3, -0.5, 0.8])
    a = angle * axis / np.linalg.norm(axis)
    np.testing.assert_allclose(oracle.rodrigues(a), Rotation.from_rotvec(a).as_matrix(), rtol=0, atol=2e-15)


def test_solve_update_matches_numpy(oracle_lib):
    """H x = -g by Cholesky == numpy.linalg.solve; pose composed on the left (R5)."""
    rng = np.random.default_rng(2)
    A = rng.standard_normal((40, 6))
    H = A.T @ A
    g = rng.standard_normal(6) * 0.01
    P = _pose(Rotation.from_rotvec([0.2, 0.1, -0.3]).as_matrix(), np.array([1.0, 2.0, 3.0]))
    st, Pn, x, th, tn = oracle.solve_update(H, g, 40, P)
    assert st == oracle.OK
    xr = np.linalg.solve(H, -g)
    np.testing.assert_allclose(x, xr, rtol=1e-12, atol=1e-15)
    dR = Rotation.from_rotvec(xr[:3]).as_matrix()
    np.testing.assert_allclose(Pn[:3, :3], dR @ P[:3, :3], atol=1e-14)
    np.testing.assert_allclose(Pn[:3, 3], dR @ P[:3, 3] + xr[3:], atol=1e-13)
    assert th == pytest.approx(np.linalg.norm(xr[:3]), rel=1e-14)


def test_degenerate_and_empty(oracle_lib):
    """SPEC.md:414 singular 6x6 (all normals parallel) -> degenerate, pose unchanged;
    SPEC.md:422/427 zero correspondences -> status, pose unchanged."""
    rng = np.random.default_rng(4)
    pts = rng.uniform(-1, 1, (500, 3)).astype(np.float32)
    pts[:, 2] = 0
    nrm = np.tile(np.array([[0, 0, 1]], np.float32), (500, 1))
    src = pts + np.array([0, 0, 0.01], np.float32)
    res = oracle.icp_run(pts, nrm, src, "point_to_plane", 5, 0.1)
    assert res.status == oracle.DEGENERATE and not res.converged
    np.testing.assert_array_equal(res.pose, np.eye(4))
    res = oracle.icp_run(pts, nrm, src + 100, "point_to_plane", 5, 0.1)
    assert res.status == oracle.NO_CORRESPONDENCES and res.n_corr == 0 and not res.converged
    np.testing.assert_array_equal(res.pose, np.eye(4))
    st, Pn, *_ = oracle.solve_update(np.eye(6), np.ones(6), 5, np.eye(4))   # count < 6
    assert st == oracle.DEGENERATE


# ----------------------------------------------------------------------------- ICP fixed points
def _kabsch(P, Q):
    """least-squares rigid R,t with Q ~ R P + t (numpy SVD with reflection fix)"""
    mp, mq = P.mean(0), Q.mean(0)
    U, S, Vt = np.linalg.svd((P - mp).T @ (Q - mq))
    D = np.diag([1, 1, np.sign(np.linalg.det(Vt.T @ U.T))])
    R = Vt.T @ D @ U.T
    return R, mq - R @ mp


def test_point_to_point_gauss_newton_converges_to_kabsch(oracle_lib):
    """DESIGN.md R6: the linearised point-to-point step iterated on fixed correspondences
    converges to the closed-form optimum (Kabsch/SVD) -- SPEC.md:404,408."""
    rng = np.random.default_rng(8)
    src = rng.uniform(-1, 1, (300, 3)).astype(np.float32)
    R0 = Rotation.from_rotvec([0.3, -0.2, 0.4]).as_matrix()
    tgt = (src @ R0.T + [0.2, -0.1, 0.3] + rng.normal(0, 0.02, (300, 3))).astype(np.float32)
    P = np.eye(4)
    corr = np.arange(300, dtype=np.int32)
    for _ in range(40):
        sys_ = oracle.icp_system_from_corr(tgt, None, src, P, "point_to_point", corr)
        st, P, *_ = oracle.solve_update(sys_.H, sys_.g, sys_.count, P)
        assert st == oracle.OK
    R, t = _kabsch(src.astype(np.float64), tgt.astype(np.float64))
    assert _rot_angle(P[:3, :3] @ R.T) < 1e-12
    np.testing.assert_allclose(P[:3, 3], t, atol=1e-12)


def test_translation_only_single_step_closed_form(oracle_lib):
    """Centred source, exact correspondences, pure translation t0: one point-to-point step
    gives alpha = 0 and tau = t0 (g = (sum s x r ; sum r) = (0 ; -m t0), H_rt = 0)."""
    rng = np.random.default_rng(9)
    src = rng.uniform(-1, 1, (256, 3))
    src -= src.mean(0)
    src = src.astype(np.float32)
    src -= src.astype(np.float64).mean(0).astype(np.float32)
    t0 = np.array([0.125, -0.25, 0.0625])
    tgt = (src.astype(np.float64) + t0).astype(np.float32)
    sys_ = oracle.icp_system_from_corr(tgt, None, src, np.eye(4), "point_to_point", np.arange(256, dtype=np.int32))
    st, P, x, *_ = oracle.solve_update(sys_.H, sys_.g, sys_.count, np.eye(4))
    assert np.abs(x[:3]).max() < 1e-6
    np.testing.assert_allclose(x[3:], t0, atol=1e-6)


def _corner_scene(rng, n_per=2000, size=0.6):
    """three orthogonal planar patches (a room corner) with analytic normals"""
    pts, nrm = [], []
    for ax in range(3):
        uv = rng.uniform(0, size, (n_per, 2))
        p = np.zeros((n_per, 3))
        others = [a for a in range(3) if a != ax]
        p[:, others[0]] = uv[:, 0]
        p[:, others[1]] = uv[:, 1]
        nn = np.zeros((n_per, 3))
        nn[:, ax] = 1.0
        pts.append(p)
        nrm.append(nn)
    return np.concatenate(pts), np.concatenate(nrm)


def test_point_to_plane_planted_motion_is_fixed_point(oracle_lib):
    """Exact correspondences on >= 3 non-parallel planes: g = 0 at the planted motion, so the
    planted pose is a fixed point of the point-to-plane step."""
    rng = np.random.default_rng(12)
    pts, nrm = _corner_scene(rng)
    tgt = pts.astype(np.float32)
    T = _pose(Rotation.from_rotvec([0.05, -0.03, 0.02]).as_matrix(), np.array([0.02, 0.01, -0.03]))
    src = ((tgt.astype(np.float64) - T[:3, 3]) @ T[:3, :3]).astype(np.float32)   # T^-1 tgt
    sys_ = oracle.icp_system_from_corr(tgt, nrm.astype(np.float32), src, T, "point_to_plane",
                                       np.arange(len(tgt), dtype=np.int32))
    st, P, x, th, tn = oracle.solve_update(sys_.H, sys_.g, sys_.count, T)
    assert th < 1e-6 and tn < 1e-6


def test_icp_recovers_planted_motion_corner(oracle_lib):
    """SPEC.md:757 / PAPER.md:195 protocol: planted 5 deg / 0.05 on a corner scene, point-to-
    plane, 15 iterations, 5 cm rejection -> rotation error < 0.1 deg, translation < 1e-3."""
    rng = np.random.default_rng(13)
    pts, nrm = _corner_scene(rng, 4000, 1.0)
    tgt = pts.astype(np.float32)
    axis = rng.standard_normal(3)
    R0 = Rotation.from_rotvec(math.radians(5) * axis / np.linalg.norm(axis)).as_matrix()
    t0 = 0.05 * np.array([1, -1, 1]) / math.sqrt(3)
    # source = target seen after the inverse motion, so the answer (source->target) is (R0, t0)
    src = ((tgt.astype(np.float64) - t0) @ R0).astype(np.float32)
    res = oracle.icp_run(tgt, nrm.astype(np.float32), src, "point_to_plane", 15, 0.05)
    assert res.status == oracle.OK
    assert math.degrees(_rot_angle(res.pose[:3, :3] @ R0.T)) < 0.1
    assert np.linalg.norm(res.pose[:3, 3] - t0) < 1e-3
    # SPEC.md:432 rmse non-increasing on a noise-free planted instance
    r = res.iter_log[:, 1]
    assert np.all(np.diff(r) <= 1e-12 + 1e-9 * r[:-1])


def test_icp_identity_converges_in_one_iteration(oracle_lib):
    """tgt = src, identity init -> converged after 1 iteration, rmse 0."""
    pts, nrm = _corner_scene(np.random.default_rng(15), 1000, 1.0)
    tgt = pts.astype(np.float32)
    for metric in ("point_to_plane", "point_to_point"):
        res = oracle.icp_run(tgt, nrm.astype(np.float32), tgt, metric, 20, 0.1, rot_tol=1e-5, trans_tol=1e-6)
        assert res.converged and res.iterations == 1 and res.rmse == 0.0 and res.n_corr == len(tgt)
        np.testing.assert_array_equal(res.pose, np.eye(4))
    # a perfect sphere with radial normals has s x n = 0: rotation unobservable -> degenerate
    w = gen.c1_sphere()
    res = oracle.icp_run(w.target, w.target_normals, w.target, "point_to_plane", 20, 0.1)
    assert res.status == oracle.DEGENERATE


def test_icp_equivariance(oracle_lib):
    """icp(Q src, Q tgt) recovers Q M Q^-1 (noise-free)."""
    rng = np.random.default_rng(14)
    pts, nrm = _corner_scene(rng, 1500, 1.0)
    R0 = Rotation.from_rotvec([0.03, 0.02, -0.04]).as_matrix()
    t0 = np.array([0.01, 0.02, -0.015])
    src = (pts - t0) @ R0
    Q = Rotation.from_rotvec([0.4, -1.1, 0.7]).as_matrix()
    qt = np.array([0.5, -0.3, 0.2])
    a = oracle.icp_run(pts.astype(np.float32), nrm.astype(np.float32), src.astype(np.float32),
                       "point_to_plane", 30, 0.1)
    b = oracle.icp_run((pts @ Q.T + qt).astype(np.float32), (nrm @ Q.T).astype(np.float32),
                       (src @ Q.T + qt).astype(np.float32), "point_to_plane", 30, 0.1)
    Tq = _pose(Q, qt)
    expect = Tq @ a.pose @ np.linalg.inv(Tq)
    assert _rot_angle(b.pose[:3, :3] @ expect[:3, :3].T) < 1e-6
    np.testing.assert_allclose(b.pose[:3, 3], expect[:3, 3], atol=1e-6)


def test_c1_sphere_translation_vs_ground_truth(oracle_lib):
    """Sanity (R19): on C1 the translation is pinned by ground truth; the rotation
    is weakly observable on a sphere and is pinned by oracle parity only."""
    w = gen.c1_sphere()
    res = oracle.icp_run(w.target, w.target_normals, w.source, "point_to_plane", 20, 0.1)
    assert res.status == oracle.OK and res.n_corr == w.n
    assert np.linalg.norm(res.pose[:3, 3] - w.gt_pose[:3, 3]) < 2e-3


def test_c4_small_lidar_vs_ground_truth(oracle_lib):
    """Sanity on a reduced LiDAR scan (8 rings x 4000 azimuths): both metrics move toward
    the planted 1.5 deg / 0.5 m motion."""
    w = gen.c4_lidar(rings=16, az=4000)
    tree = oracle.KDTree(w.target)
    res = oracle.icp_run(None, w.target_normals, w.source, "point_to_plane", 50, 1.0, tree=tree)
    assert res.status == oracle.OK
    err_t = np.linalg.norm(res.pose[:3, 3] - w.gt_pose[:3, 3])
    err_r = math.degrees(_rot_angle(res.pose[:3, :3] @ w.gt_pose[:3, :3].T))
    assert err_t < 0.1 and err_r < 0.2, (err_t, err_r)


# ----------------------------------------------------------------------------- PCA normals
def test_pca_normals_plane_and_orientation(oracle_lib):
    """SPEC.md:236 planar case: every normal equals the plane normal, oriented to the viewpoint."""
    g = np.stack(np.meshgrid(np.arange(30), np.arange(30), indexing="ij"), -1).reshape(-1, 2) * 0.01
    pts = np.concatenate([g, np.zeros((len(g), 1))], 1).astype(np.float32)
    n_up, curv = oracle.pca_normals(pts, 10, view=(0, 0, 1))
    np.testing.assert_allclose(n_up, np.tile([0, 0, 1], (len(pts), 1)), atol=1e-9)
    assert np.abs(curv).max() < 1e-12
    n_dn, _ = oracle.pca_normals(pts, 10, view=(0, 0, -1))
    np.testing.assert_allclose(n_dn, np.tile([0, 0, -1], (len(pts), 1)), atol=1e-9)


def test_pca_normals_match_numpy_eigh(oracle_lib):
    """Per-point PCA over the 10-NN (found by scipy cKDTree) with numpy eigh."""
    rng = np.random.default_rng(21)
    pts = rng.standard_normal((3000, 3))
    pts = (pts / np.linalg.norm(pts, axis=1, keepdims=True) + rng.normal(0, 0.01, (3000, 3))).astype(np.float32)
    nrm, curv = oracle.pca_normals(pts, 10, view=(0, 0, 0))
    _, nb = cKDTree(pts.astype(np.float64)).query(pts.astype(np.float64), k=10)
    P = pts.astype(np.float64)[nb]
    Cv = np.einsum("nki,nkj->nij", P - P.mean(1, keepdims=True), P - P.mean(1, keepdims=True)) / 10
    w, V = np.linalg.eigh(Cv)
    ref = V[:, :, 0]
    ref *= np.where(np.einsum("ni,ni->n", -pts.astype(np.float64), ref) < 0, -1, 1)[:, None]
    # angle from the cross product of the renormalised normals (robust near 0)
    nn = nrm.astype(np.float64) / np.linalg.norm(nrm.astype(np.float64), axis=1, keepdims=True)
    ang = np.arcsin(np.clip(np.linalg.norm(np.cross(nn, ref), axis=1), 0, 1))
    assert np.quantile(ang, 0.999) < 1e-6
    np.testing.assert_allclose(curv, w[:, 0] / w.sum(1), atol=1e-6)
    # orientation toward the viewpoint (origin)
    assert (np.einsum("ni,ni->n", -pts.astype(np.float64), nrm.astype(np.float64)) >= -1e-7).all()


@pytest.mark.parametrize("w", [(1.0, 0.0), (0.0, 1.0)])
def test_combined_reduces_to_single_metrics(oracle_lib, w):
    """SURVEY.md 8(f) NEXT-1 pin: weights (1,0) and (0,1) give the point-to-point and the
    point-to-plane systems exactly (same correspondences, same ICP trajectory)."""
    rng = np.random.default_rng(5)
    tgt = rng.uniform(-1, 1, (400, 3)).astype(np.float32)
    nrm = rng.standard_normal((400, 3))
    nrm = (nrm / np.linalg.norm(nrm, axis=1, keepdims=True)).astype(np.float32)
    src = (tgt + rng.normal(0, 0.01, tgt.shape)).astype(np.float32)
    pose = _pose(Rotation.from_rotvec([0.02, 0.01, -0.03]).as_matrix(), np.array([0.01, -0.02, 0.0]))
    oracle.set_combined_weights(*w)
    single = "point_to_point" if w[0] == 1.0 else "point_to_plane"
    a = oracle.icp_system(tgt, nrm, src, pose, "combined", 0.2)
    b = oracle.icp_system(tgt, nrm, src, pose, single, 0.2)
    np.testing.assert_array_equal(a.H, b.H)
    np.testing.assert_array_equal(a.g, b.g)
    assert a.sse == b.sse and a.count == b.count
