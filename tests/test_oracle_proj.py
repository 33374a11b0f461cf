"""Pins for the projective data-association oracle (oracle.proj_system / proj_run;
SURVEY.md 8(f) NEXT-2, PAPER.md:83 / PAPER.md:140, DESIGN.md
readings R23-R26) against things other than itself: integer closed forms of the pixel
lookup, hand-built rounding / bounds / validity / rejection cases, an independent numpy
recomputation of the normal equations, the fixed point and a planted motion.  CPU only.
"""
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import gen
import oracle
from tests.workloads import c3, rot_angle


def _plane_image(w, h, fx, fy, cx, cy, z):
    """organised cloud of the fronto-parallel plane at depth z (row-major pixels)"""
    u, v = np.meshgrid(np.arange(w, dtype=np.float64), np.arange(h, dtype=np.float64))
    zz = np.full(u.shape, z)
    return np.stack([(u - cx) * zz / fx, (v - cy) * zz / fy, zz], -1).reshape(-1, 3).astype(np.float32)


def _pose(R=np.eye(3), t=np.zeros(3)):
    T = np.eye(4)
    T[:3, :3] = R
    T[:3, 3] = t
    return T


INTR_SMALL = (16, 12, 20.0, 20.0, 7.5, 5.5)


def test_identity_pairs_every_point_with_itself():
    """SPEC.md:397 example: src = the valid target points of an organised cloud -> every point
    pairs with itself at distance 0 (here the C3 frame, with a block of invalid pixels)"""
    w = c3()
    tgt = w.target.copy()
    bad = np.zeros(tgt.shape[0], bool)
    bad[1000:1500] = True
    bad[::97] = True
    tgt[bad, 2] = 0.0                                   # invalid pixels (z <= 0)
    tgt[5, :] = np.nan                                  # and a non-finite one
    bad[5] = True
    s = oracle.proj_system(tgt, None, (640, 480, gen.FX, gen.FY, gen.CX, gen.CY), tgt, np.eye(4),
                           "point_to_point", 0.05)
    want = np.where(bad, -1, np.arange(tgt.shape[0]))
    np.testing.assert_array_equal(s.corr_idx, want)
    assert np.all(s.corr_d2[~bad] == 0.0) and np.all(np.isinf(s.corr_d2[bad]))
    assert s.count == int((~bad).sum()) and s.sse == 0.0


@pytest.mark.parametrize("axis", [0, 1])
def test_one_pixel_shift_closed_form(axis):
    """translating a fronto-parallel plane at depth Z by Z/f along x (y) moves every pixel's
    projection by exactly one column (row): pixel k pairs with k - 1 (k - w); the first
    column (row) projects out of bounds and the pairs coincide (d^2 = 0 up to fp32 inputs).  Pins the row-major index v*w + u, the u/v roles and
    the projection formula."""
    w, h, fx, fy, cx, cy = INTR_SMALL
    Z = 2.0
    pts = _plane_image(w, h, fx, fy, cx, cy, Z)
    t = np.zeros(3)
    t[axis] = -Z / (fx if axis == 0 else fy)
    s = oracle.proj_system(pts, None, INTR_SMALL, pts, _pose(t=t), "point_to_point", 1.0)
    k = np.arange(w * h)
    u, v = k % w, k // w
    if axis == 0:
        want = np.where(u >= 1, k - 1, -1)
    else:
        want = np.where(v >= 1, k - w, -1)
    np.testing.assert_array_equal(s.corr_idx, want)
    ok = want >= 0
    assert np.all(s.corr_d2[ok] < 1e-12)              # s = p + t IS the shifted pixel's point


def test_rounding_half_away_from_zero_and_bounds():
    """round half away from zero, THEN the bounds check (R24):
    u = 0.5 -> 1 (half-to-even would give 0), 2.5 -> 3, -0.5 -> -1 (out of bounds; half-to-even
    would give pixel 0), 3.5 = w - 0.5 -> 4 = w (out of bounds)."""
    w, h = 4, 1
    intr = (w, h, 1.0, 1.0, 0.0, 0.0)               # u = x / z, v = y / z
    src = np.array([[0.5, 0.0, 1.0], [2.5, 0.0, 1.0], [-0.5, 0.0, 1.0], [3.5, 0.0, 1.0],
                    [1.4999999, 0.0, 1.0], [0.0, 0.5, 1.0], [0.0, -0.4, 1.0]], np.float32)
    tgt = np.array([[0.0, 0.0, 1.0], [0.5, 0.0, 1.0], [1.5, 0.0, 1.0], [2.5, 0.0, 1.0]], np.float32)
    s = oracle.proj_system(tgt, None, intr, src, np.eye(4), "point_to_point", 10.0)
    np.testing.assert_array_equal(s.corr_idx, [1, 3, -1, -1, 1, -1, 0])
    np.testing.assert_array_equal(s.uv[:4, 0], [0.5, 2.5, -0.5, 3.5])


def test_behind_camera_invalid_and_rejection_boundary():
    """s_z <= 0 -> no pair; invalid target pixel -> no pair; |s - t| == max_dist is accepted
    (inclusive, R2) and a hair beyond is rejected."""
    intr = (1, 1, 1.0, 1.0, 0.0, 0.0)
    tgt = np.array([[0.0, 0.0, 1.5]], np.float32)
    src = np.array([[0.0, 0.0, 1.0], [0.0, 0.0, -1.0], [0.0, 0.0, 0.0], [0.2, 0.0, 1.5]], np.float32)
    s = oracle.proj_system(tgt, None, intr, src, np.eye(4), "point_to_point", 0.5)
    np.testing.assert_array_equal(s.corr_idx, [0, -1, -1, 0])   # (0.2 / 1.5, 0) rounds to pixel 0
    assert s.corr_d2[0] == 0.25
    s2 = oracle.proj_system(tgt, None, intr, src[:1], np.eye(4), "point_to_point", 0.4999999)
    assert s2.corr_idx[0] == -1 and s2.count == 0
    bad = tgt.copy()
    bad[0, 2] = -1.0
    s3 = oracle.proj_system(bad, None, intr, src[:1], np.eye(4), "point_to_point", 10.0)
    assert s3.corr_idx[0] == -1


@pytest.mark.parametrize("metric", ["point_to_plane", "point_to_point"])
def test_system_matches_numpy_dense_recomputation(metric):
    """H = sum J^T J, g = sum J^T r over the projective pairs, recomputed with dense numpy
    from the pixel indices derived independently with numpy (np.round is half-to-even, so
    points within 1e-6 of a half-pixel are excluded from the index comparison)."""
    w = c3()
    intr = (640, 480, gen.FX, gen.FY, gen.CX, gen.CY)
    P = _pose(Rotation.from_rotvec([0.004, -0.003, 0.0175]).as_matrix(), np.array([0.01, -0.02, 0.015]))
    sub = w.source[::7]
    sy = oracle.proj_system(w.target, w.target_normals, intr, sub, P, metric, 0.05)
    S = sub.astype(np.float64) @ P[:3, :3].T + P[:3, 3]
    uf = gen.FX * S[:, 0] / S[:, 2] + gen.CX
    vf = gen.FY * S[:, 1] / S[:, 2] + gen.CY
    ui, vi = np.floor(uf + 0.5).astype(np.int64), np.floor(vf + 0.5).astype(np.int64)
    inb = (S[:, 2] > 0) & (ui >= 0) & (ui < 640) & (vi >= 0) & (vi < 480)
    k = np.where(inb, vi * 640 + ui, 0)
    T = w.target.astype(np.float64)[k]
    d2 = ((S - T) ** 2).sum(1)
    acc = inb & (d2 <= 0.05 ** 2)
    near_half = (np.abs(uf - np.floor(uf) - 0.5) < 1e-6) | (np.abs(vf - np.floor(vf) - 0.5) < 1e-6)
    want = np.where(acc, k, -1)
    assert np.array_equal(sy.corr_idx[~near_half], want[~near_half])
    sel = sy.corr_idx >= 0
    s_, t_ = S[sel], w.target.astype(np.float64)[sy.corr_idx[sel]]
    if metric == "point_to_plane":
        n_ = w.target_normals.astype(np.float64)[sy.corr_idx[sel]]
        J = np.concatenate([np.cross(s_, n_), n_], 1)
        r = ((s_ - t_) * n_).sum(1)
        H, g = J.T @ J, J.T @ r
    else:
        n = len(s_)
        Sx = np.zeros((n, 3, 3))                       # [s]x
        Sx[:, 0, 1], Sx[:, 0, 2] = -s_[:, 2], s_[:, 1]
        Sx[:, 1, 0], Sx[:, 1, 2] = s_[:, 2], -s_[:, 0]
        Sx[:, 2, 0], Sx[:, 2, 1] = -s_[:, 1], s_[:, 0]
        J = np.concatenate([-Sx, np.broadcast_to(np.eye(3), (n, 3, 3))], 2)   # [-[s]x, I3]
        H = np.einsum("nai,naj->ij", J, J)
        g = np.einsum("nai,na->i", J, s_ - t_)
    assert sy.count == int(sel.sum())
    np.testing.assert_allclose(sy.H, H, rtol=1e-10, atol=1e-10 * np.abs(H).max())
    np.testing.assert_allclose(sy.g, g, rtol=1e-9, atol=1e-10 * sy.gabs.max())


def test_proj_system_equals_given_correspondence_system():
    """the accumulation is the plain definition over the pairs the engine found (the same
    numbers as the kd-tree path's accumulation of GIVEN correspondences)"""
    w = c3()
    intr = (640, 480, gen.FX, gen.FY, gen.CX, gen.CY)
    sy = oracle.proj_system(w.target, w.target_normals, intr, w.source, np.eye(4), "point_to_plane", 0.05)
    sc = oracle.icp_system_from_corr(w.target, w.target_normals, w.source, np.eye(4), "point_to_plane",
                                     sy.corr_idx.astype(np.int32))
    assert sc.count == sy.count
    np.testing.assert_array_equal(sc.H, sy.H)
    np.testing.assert_array_equal(sc.g, sy.g)


def test_run_identity_fixed_point():
    """source = target, pose I: every residual is 0, so g = 0, x = 0 and the pose stays I
    exactly (the planted-motion fixed point)"""
    w = c3()
    intr = (640, 480, gen.FX, gen.FY, gen.CX, gen.CY)
    r = oracle.proj_run(w.target, w.target_normals, intr, w.target, "point_to_plane", 3, 0.05)
    assert r.status == 0
    np.testing.assert_array_equal(r.pose, np.eye(4))
    assert r.rmse == 0.0 and r.n_corr == w.n


def test_run_recovers_c3_planted_motion():
    """C3 (3 deg / 3 cm camera motion): projective ICP started at the ground truth stays
    there (0.05 deg / 2 mm), and from the identity it reaches it (projective association
    converges far more slowly than exact NN, R26: 300 iterations)"""
    w = c3()
    intr = (640, 480, gen.FX, gen.FY, gen.CX, gen.CY)

    def err(P):
        E = P @ np.linalg.inv(w.gt_pose)
        return math.degrees(rot_angle(E[:3, :3])), float(np.linalg.norm(E[:3, 3]))
    r = oracle.proj_run(w.target, w.target_normals, intr, w.source, "point_to_plane", 10, 0.05, pose_init=w.gt_pose)
    a, t = err(r.pose)
    assert a < 0.05 and t < 2e-3
    r = oracle.proj_run(w.target, w.target_normals, intr, w.source, "point_to_plane", 300, 0.05)
    a, t = err(r.pose)
    assert a < 0.05 and t < 2e-3
    a0, t0 = err(np.eye(4))
    assert a0 > 2.5 and t0 > 0.02
