"""GPU parity: the CUDA path (through the C ABI) against the fp64 CPU oracle on the same
seeded inputs.  Tolerances are BASELINE.json north_star's:
  * NN indices bit-exact wherever (d2_2nd - d2_best) > 1e-6 * d2_best (else the GPU's pick
    must itself be within the near-tie band), NN d^2 within 1e-6 relative;
  * rejection decisions equal outside the ambiguous band |d^2/max^2 - 1| <= 2e-6 (R2);
  * H within 1e-5 relative Frobenius, g within 1e-5 of ||g|| (or of ||sum|J r|||, R16),
    also after reconciling near-tie flips through the GPU's own correspondences (R17);
  * final poses within 1e-4 rad and 1e-5 units.
"""
import math

import numpy as np
import pytest
import torch

import gen
import oracle
from tests import workloads as W

pytestmark = pytest.mark.gpu

NN_REL = 1e-6
BAND = 2e-6


@pytest.fixture(scope="module")
def cil():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1807_00399_b200 as cil
    return cil


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a)).cuda()


def check_nn(tgt, queries_f64, g_idx, g_d2, o_idx, o_d2, max_d2=math.inf):
    """GPU NN (g_*) vs oracle k=2 NN (o_* [m,2]) with the north_star masks."""
    g_idx = np.asarray(g_idx, np.int64)
    g_d2 = np.asarray(g_d2, np.float64)
    d1, d2nd = o_d2[:, 0], o_d2[:, 1]
    o_acc = o_idx[:, 0] >= 0
    g_acc = g_idx >= 0
    band = np.isfinite(max_d2) & (np.abs(d1 / max_d2 - 1.0) <= BAND) if np.isfinite(max_d2) else np.zeros(len(d1), bool)
    mism = (o_acc != g_acc) & ~band
    assert not mism.any(), f"{mism.sum()} rejection decisions differ outside the band"
    both = o_acc & g_acc
    # distances within 1e-6 relative (exact zero stays zero)
    err = np.abs(g_d2[both] - d1[both])
    assert (err <= NN_REL * d1[both]).all(), f"max rel d2 err {np.max(err / np.maximum(d1[both], 1e-300))}"
    # indices bit-exact outside the near-tie band
    with np.errstate(invalid="ignore"):
        clear = both & ~(d2nd - d1 <= NN_REL * d1)      # inf - inf (no 2nd point) counts as clear
    bad = clear & (g_idx != o_idx[:, 0])
    assert not bad.any(), f"{bad.sum()} NN indices differ with a clear gap"
    # inside the band the GPU's pick must itself be a near-tie (fp64 distance of its pick)
    tie = both & ~clear & (g_idx != o_idx[:, 0])
    if tie.any():
        q = queries_f64[tie]
        t = tgt[g_idx[tie]].astype(np.float64)
        dd = ((q - t) ** 2).sum(1)
        assert (dd <= d1[tie] * (1 + 2 * NN_REL) + 0.0).all()
    return int(clear.sum()), int(tie.sum())


# ------------------------------------------------------------------ NN
INDEXES = ["bvh", "grid"]


@pytest.mark.parametrize("index", INDEXES)
@pytest.mark.parametrize("n,m,leaf", [(1, 5, 8), (7, 33, 8), (8, 64, 8), (9, 257, 4), (1000, 1000, 16),
                                      (4097, 3001, 32), (65537, 100003, 8)])
def test_nn_small_ragged(cil, n, m, leaf, index):
    rng = np.random.default_rng(n + m)
    T = rng.standard_normal((n, 3)).astype(np.float32)
    Q = (rng.standard_normal((m, 3)) * 1.1).astype(np.float32)
    t = cil.cil_target_build(dev(T), None, leaf_size=leaf, index=index)
    gi, gd = cil.cil_nn_query(t, dev(Q))
    o_idx, o_d2 = oracle.knn(T, Q.astype(np.float64), k=2)
    check_nn(T, Q.astype(np.float64), gi.cpu().numpy(), gd.cpu().numpy(), o_idx, o_d2)
    info = t.info()
    assert info.n == n and info.leaf_size == leaf and info.n_leaves == (n + leaf - 1) // leaf


@pytest.mark.parametrize("n", [257, 2049, 8193, 16385, 32769, 131073])
def test_nn_build_sort_tile_regimes(cil, n):
    """index builds on both sides of every small-input sort-tile size and scan path (and of the
    programmatic-dependent-launch threshold, 32,768 points): every query against the oracle"""
    rng = np.random.default_rng(n)
    T = rng.standard_normal((n, 3)).astype(np.float32)
    Q = (rng.standard_normal((4001, 3)) * 1.1).astype(np.float32)
    t = cil.cil_target_build(dev(T), None)
    gi, gd = cil.cil_nn_query(t, dev(Q))
    o_idx, o_d2 = oracle.knn(T, Q.astype(np.float64), k=2)
    check_nn(T, Q.astype(np.float64), gi.cpu().numpy(), gd.cpu().numpy(), o_idx, o_d2)


@pytest.mark.parametrize("index", INDEXES)
def test_nn_ties_lowest_original_index(cil, index):
    """R1: exact ties (duplicated integer grid points, cube centres) -> lowest original index."""
    g = np.stack(np.meshgrid(*[np.arange(10)] * 3, indexing="ij"), -1).reshape(-1, 3).astype(np.float32)
    T = np.concatenate([g[::-1], g, g[::-1]])
    Q = np.concatenate([g, g + 0.5, g + 0.25, g - 0.5]).astype(np.float32)
    t = cil.cil_target_build(dev(T), None, leaf_size=4, index=index)
    gi, gd = cil.cil_nn_query(t, dev(Q))
    from scipy.spatial.distance import cdist
    D = cdist(Q.astype(np.float64), T.astype(np.float64), "sqeuclidean")
    ref = np.argmin(D, 1)
    assert np.array_equal(gi.cpu().numpy(), ref)
    assert np.array_equal(gd.cpu().numpy().astype(np.float64), D[np.arange(len(Q)), ref])


@pytest.mark.parametrize("index", INDEXES)
def test_nn_bounded_and_empty(cil, index):
    rng = np.random.default_rng(1)
    T = rng.random((5000, 3)).astype(np.float32)
    Q = rng.random((7000, 3)).astype(np.float32)
    t = cil.cil_target_build(dev(T), None, index=index)
    for md in (0.0, 0.01, 0.03):
        gi, gd = cil.cil_nn_query(t, dev(Q), max_dist=md)
        o_idx, o_d2 = oracle.knn(T, Q.astype(np.float64), k=2, max_dist=md)
        check_nn(T, Q.astype(np.float64), gi.cpu().numpy(), gd.cpu().numpy(), o_idx, o_d2,
                 max_d2=float(np.float32(md) ** 2) if md > 0 else 0.0)
    # empty query set
    gi, gd = cil.cil_nn_query(t, torch.empty((0, 3), device="cuda"))
    assert gi.numel() == 0
    # self query -> itself at distance 0
    gi, gd = cil.cil_nn_query(t, dev(T))
    assert np.array_equal(gi.cpu().numpy(), np.arange(5000)) and (gd.cpu().numpy() == 0).all()


@pytest.mark.parametrize("shape", ["point", "line", "plane", "far", "lidar_like"])
def test_nn_grid_degenerate(cil, shape):
    """The uniform grid on degenerate extents (all points equal, a line, a plane: flat axes get
    one cell), queries far outside the bounding box (shells never reach: BVH fallback) and a
    strongly non-uniform cloud -- against the oracle, both indexes."""
    rng = np.random.default_rng(11)
    n, m = 3000, 4000
    if shape == "point":
        T = np.tile(np.float32([[1.5, -2.0, 3.25]]), (n, 1))
        Q = (rng.standard_normal((m, 3)) + [1.5, -2.0, 3.25]).astype(np.float32)
    elif shape == "line":
        T = np.stack([rng.random(n), np.zeros(n), np.zeros(n)], 1).astype(np.float32)
        Q = rng.random((m, 3)).astype(np.float32)
    elif shape == "plane":
        T = np.stack([rng.random(n), rng.random(n), np.full(n, 0.5)], 1).astype(np.float32)
        Q = rng.random((m, 3)).astype(np.float32)
    elif shape == "far":
        T = rng.random((n, 3)).astype(np.float32)
        Q = (rng.standard_normal((m, 3)) * 50.0).astype(np.float32)
    else:
        r = np.exp(rng.uniform(0, 4, n))
        a = rng.uniform(0, 2 * np.pi, n)
        T = np.stack([r * np.cos(a), r * np.sin(a), rng.normal(0, 0.01, n)], 1).astype(np.float32)
        Q = (T[rng.integers(0, n, m)] + rng.normal(0, 0.05, (m, 3))).astype(np.float32)
    o_idx, o_d2 = oracle.knn(T, Q.astype(np.float64), k=2)
    res = []
    for index in INDEXES:
        t = cil.cil_target_build(dev(T), None, index=index)
        gi, gd = cil.cil_nn_query(t, dev(Q))
        check_nn(T, Q.astype(np.float64), gi.cpu().numpy(), gd.cpu().numpy(), o_idx, o_d2)
        assert t.info().index_kind == (cil.CIL_INDEX_GRID if index == "grid" else cil.CIL_INDEX_BVH)
        res.append((gi.cpu().numpy(), gd.cpu().numpy()))
    # both indexes return the same (exact) minimum of the same fp32 arithmetic
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])


@pytest.mark.parametrize("index", INDEXES)
def test_nn_c2_full_size(cil, index):
    """BASELINE.json configs[1] at full size (2^20 x 2^20), every query checked."""
    w = W.c2()
    t = cil.cil_target_build(dev(w.target), None, index=index)
    gi, gd = cil.cil_nn_query(t, dev(w.source))
    torch.cuda.synchronize()
    o_idx, o_d2 = oracle.knn(None, w.source.astype(np.float64), k=2, tree=W.oracle_tree(w))
    clear, tie = check_nn(w.target, w.source.astype(np.float64), gi.cpu().numpy(), gd.cpu().numpy(), o_idx, o_d2)
    assert clear >= w.m - 50


# ------------------------------------------------------------------ one iteration
def _pose(R=np.eye(3), t=np.zeros(3)):
    T = np.eye(4)
    T[:3, :3] = R
    T[:3, 3] = t
    return T


def _perturb(gt, frac):
    """pose `frac` of the way from identity to ground truth"""
    from scipy.spatial.transform import Rotation
    rv = Rotation.from_matrix(gt[:3, :3]).as_rotvec() * frac
    return _pose(Rotation.from_rotvec(rv).as_matrix(), gt[:3, 3] * frac)


COMBINED_W = (0.4, 1.3)   # weights of the combined metric in these tests


def _params(cil, metric, iters, max_dist):
    if metric == "combined":
        oracle.set_combined_weights(*COMBINED_W)
        return cil.make_params(metric, iters, max_dist, w_point=COMBINED_W[0], w_plane=COMBINED_W[1])
    return cil.make_params(metric, iters, max_dist)


def check_iteration(cil, w, pose, metric, tree=None, sample=None, leaf=0, index="bvh"):
    """cil_icp_iterate vs oracle at the same pose_in: correspondences, H, g, pose_out."""
    t = cil.cil_target_build(dev(w.target), dev(w.target_normals) if w.target_normals is not None else None,
                             leaf_size=leaf, index=index)
    prm = _params(cil, metric, 1, w.max_dist)
    P = dev(pose.astype(np.float64))
    pose_out, sys_t, ci, cd = cil.cil_icp_iterate(t, dev(w.source), P, prm, want_corr=True)
    gs = cil.decode_system(sys_t)
    g_idx = ci.cpu().numpy()
    g_d2 = cd.cpu().numpy()
    tree = tree or W.oracle_tree(w)
    o = oracle.icp_system(None, w.target_normals, w.source, pose, metric, w.max_dist, tree=tree)
    s64 = oracle.transform(pose, w.source)
    o_idx = np.stack([o.corr_idx, np.where(np.isfinite(o.corr_d2nd), 0, -1)], 1)
    o_d2 = np.stack([o.corr_d2, o.corr_d2nd], 1)
    check_nn(w.target, s64, g_idx, g_d2, o_idx, o_d2, max_d2=w.max_dist ** 2)
    # H, g against the oracle's own system (R16) ...
    assert gs.status == cil.CIL_OK
    assert abs(gs.n_corr - o.count) <= max(2, 1e-5 * o.count)
    relH = np.linalg.norm(gs.H - o.H) / np.linalg.norm(o.H)
    gscale = max(np.linalg.norm(o.g), 1e-3 * np.linalg.norm(o.gabs))
    relg = np.linalg.norm(gs.g - o.g) / gscale
    assert relH <= 1e-5 and relg <= 1e-5, (relH, relg)
    # ... and reconciled through the GPU's own correspondences (R17): much tighter
    r = oracle.icp_system_from_corr(w.target, w.target_normals, w.source, pose, metric, g_idx.astype(np.int32))
    assert r.count == gs.n_corr
    relH2 = np.linalg.norm(gs.H - r.H) / np.linalg.norm(r.H)
    relg2 = np.linalg.norm(gs.g - r.g) / max(np.linalg.norm(r.g), 1e-3 * np.linalg.norm(r.gabs))
    assert relH2 <= 1e-6 and relg2 <= 1e-5, (relH2, relg2)
    # pose_out: the oracle's solve/update of the GPU's own (H, g) ...
    st, Pr, x, _, _ = oracle.solve_update(gs.H, gs.g, gs.n_corr, pose)
    Pg = pose_out.cpu().numpy()
    assert W.rot_angle(Pg[:3, :3] @ Pr[:3, :3].T) < 1e-12 and np.abs(Pg[:3, 3] - Pr[:3, 3]).max() < 1e-12
    # ... and the oracle's full step
    st, Po, *_ = oracle.solve_update(o.H, o.g, o.count, pose)
    assert W.rot_angle(Pg[:3, :3] @ Po[:3, :3].T) < 1e-4 and np.abs(Pg[:3, 3] - Po[:3, 3]).max() < 1e-5
    return gs, g_idx


@pytest.mark.parametrize("frac", [0.0, 0.7])
def test_iterate_c1(cil, frac):
    w = W.c1()
    check_iteration(cil, w, _perturb(w.gt_pose, frac), "point_to_plane")


@pytest.mark.parametrize("metric", ["point_to_plane", "point_to_point", "combined"])
def test_iterate_c4_reduced(cil, metric):
    w = W.c4("point_to_plane" if metric == "combined" else metric, rings=16, az=8000)
    for frac in (0.0, 0.5, 1.0):
        check_iteration(cil, w, _perturb(w.gt_pose, frac), metric)


@pytest.mark.parametrize("logn", [16, 18, 20])
def test_iterate_c5(cil, logn):
    w = W.c5(logn)
    check_iteration(cil, w, np.eye(4), "point_to_plane")


@pytest.mark.parametrize("case", ["c1", "c4", "c5", "c3"])
def test_iterate_grid_index(cil, case):
    """The stateless iterate on the uniform-grid index (CIL_INDEX_GRID) against the oracle, and
    bit-equal to the BVH path (both return the exact minimum of the same fp32 arithmetic; the
    accumulation is the same kernel)."""
    if case == "c1":
        w, poses = W.c1(), None
    elif case == "c4":
        w, poses = W.c4("point_to_plane", rings=16, az=8000), None
    elif case == "c5":
        w, poses = W.c5(16), [np.eye(4)]
    else:
        w, poses = W.c3(), [np.eye(4)]
    poses = poses or [_perturb(w.gt_pose, f) for f in (0.0, 0.5, 1.0)]
    tree = W.oracle_tree(w)
    for pose in poses:
        gs, gi = check_iteration(cil, w, pose, "point_to_plane", tree=tree, index="grid")
        bs, bi = check_iteration(cil, w, pose, "point_to_plane", tree=tree, index="bvh")
        assert np.array_equal(gi, bi)
        assert np.array_equal(gs.H, bs.H) and np.array_equal(gs.g, bs.g)


def test_iterate_c3(cil):
    w = W.c3()
    check_iteration(cil, w, np.eye(4), "point_to_plane")


@pytest.mark.parametrize("leaf", [4, 16, 32])
def test_iterate_leaf_sizes(cil, leaf):
    w = W.c4("point_to_plane", rings=8, az=6000)
    check_iteration(cil, w, _perturb(w.gt_pose, 0.3), "point_to_plane", leaf=leaf)


# ------------------------------------------------------------------ the loop
def check_run(cil, w, metric, leaf=0):
    t = cil.cil_target_build(dev(w.target), dev(w.target_normals) if w.target_normals is not None else None,
                             leaf_size=leaf)
    prm = _params(cil, metric, w.max_iters, w.max_dist)
    res_t, log = cil.cil_icp_run(t, dev(w.source), dev(np.eye(4)), prm)
    res = cil.decode_result(res_t)
    o = oracle.icp_run(None, w.target_normals, w.source, metric, w.max_iters, w.max_dist, tree=W.oracle_tree(w))
    assert res.status == o.status == cil.CIL_OK
    assert res.iterations == o.iterations == w.max_iters
    dr = W.rot_angle(res.pose[:3, :3] @ o.pose[:3, :3].T)
    dt = np.abs(res.pose[:3, 3] - o.pose[:3, 3]).max()
    assert dr <= 1e-4 and dt <= 1e-5, (dr, dt)
    lg = log.cpu().numpy()
    np.testing.assert_allclose(lg[:, 0], o.iter_log[:, 0], rtol=1e-4, atol=3)
    # rmse: a near-tie or rejection-band flip swaps a pair's plane residual outright, so the
    # per-iteration rmse agrees to ~1e-4 relative, not to the pose tolerance
    np.testing.assert_allclose(lg[:, 1], o.iter_log[:, 1], rtol=1e-3)
    # the loop equals the chain of stateless iterations bit for bit (warm start is exact)
    P = dev(np.eye(4))
    for _ in range(w.max_iters):
        P, *_ = cil.cil_icp_iterate(t, dev(w.source), P, prm, want_sys=False)
    assert np.array_equal(P.cpu().numpy(), res.pose)
    return res, o


def test_run_c1(cil):
    check_run(cil, W.c1(), "point_to_plane")


@pytest.mark.parametrize("metric", ["point_to_plane", "point_to_point", "combined"])
def test_small_path_equals_tree_path(cil, metric):
    """C1 (4,096 points) takes the small-problem path (brute-force exact NN staged in shared
    memory, one cooperative launch for the run); with it disabled (debug bit 6) the BVH
    engine runs.  Both must return the same exact correspondences (bit-equal, no near ties
    here) and systems equal up to the summation order; run poses within 1e-9."""
    w = W.c1()
    prm = _params(cil, metric, w.max_iters, w.max_dist)
    prm1 = _params(cil, metric, 1, w.max_dist)
    out = []
    try:
        for flags in (0, 64):
            cil.set_debug_flags(flags)
            t = cil.cil_target_build(dev(w.target), dev(w.target_normals))
            P = dev(_perturb(w.gt_pose, 0.3))
            pose_out, sys_t, ci, cd = cil.cil_icp_iterate(t, dev(w.source), P, prm1, want_corr=True)
            res_t, log = cil.cil_icp_run(t, dev(w.source), dev(np.eye(4)), prm)
            out.append((ci.cpu().numpy(), cd.cpu().numpy(), cil.decode_system(sys_t), cil.decode_result(res_t),
                        log.cpu().numpy()))
    finally:
        cil.set_debug_flags(0)
    (ia, da, sa, ra, la), (ib, db, sb, rb, lb) = out
    assert np.array_equal(ia, ib) and np.array_equal(da, db)
    # (fp32 per-thread sums grouped differently: ~1e-8 relative)
    assert sa.n_corr == sb.n_corr and np.linalg.norm(sa.H - sb.H) <= 1e-6 * np.linalg.norm(sb.H)
    assert np.linalg.norm(sa.g - sb.g) <= 1e-5 * max(np.linalg.norm(sb.g), 1e-12)
    assert ra.status == rb.status == 0 and ra.iterations == rb.iterations
    assert W.rot_angle(ra.pose[:3, :3] @ rb.pose[:3, :3].T) <= 1e-6 and np.abs(ra.pose[:3, 3] - rb.pose[:3, 3]).max() <= 1e-7
    np.testing.assert_array_equal(la[:, 0], lb[:, 0])


@pytest.mark.parametrize("n,m", [(1, 1), (7, 100), (300, 37), (8192, 8000), (2000, 33000)])
def test_small_path_ragged(cil, n, m):
    """ragged small problems (one target point, more/less sources than targets, a group size
    of 1..32 lanes per query, the largest staged target) against the oracle's iteration"""
    rng = np.random.default_rng(n * 7 + m)
    T = rng.standard_normal((n, 3)).astype(np.float32)
    N = rng.standard_normal((n, 3))
    N = (N / np.linalg.norm(N, axis=1, keepdims=True)).astype(np.float32)
    S = (T[rng.integers(0, n, m)] + rng.normal(0, 0.05, (m, 3))).astype(np.float32)
    t = cil.cil_target_build(dev(T), dev(N))
    prm = cil.make_params("point_to_plane", 1, 0.2)
    pose_out, sys_t, ci, cd = cil.cil_icp_iterate(t, dev(S), dev(np.eye(4)), prm, want_corr=True)
    o = oracle.icp_system(T, N, S, np.eye(4), "point_to_plane", 0.2)
    o_idx = np.stack([o.corr_idx, np.where(np.isfinite(o.corr_d2nd), 0, -1)], 1)
    o_d2 = np.stack([o.corr_d2, o.corr_d2nd], 1)
    check_nn(T, S.astype(np.float64), ci.cpu().numpy(), cd.cpu().numpy(), o_idx, o_d2, max_d2=0.04)
    gs = cil.decode_system(sys_t)
    r = oracle.icp_system_from_corr(T, N, S, np.eye(4), "point_to_plane", ci.cpu().numpy().astype(np.int32))
    assert r.count == gs.n_corr
    if r.count:
        assert np.linalg.norm(gs.H - r.H) <= 1e-6 * np.linalg.norm(r.H)


@pytest.mark.parametrize("metric", ["point_to_plane", "point_to_point", "combined"])
def test_run_c4_reduced(cil, metric):
    check_run(cil, W.c4("point_to_plane" if metric == "combined" else metric, rings=16, az=8000), metric)


@pytest.mark.parametrize("w", [(1.0, 0.0), (0.0, 1.0)])
def test_combined_reduces_to_single_metrics_gpu(cil, w):
    """NEXT-1 pin on the GPU path: combined (1,0) / (0,1) runs end at the single-metric poses."""
    wl = W.c4("point_to_plane", rings=8, az=4000)
    t = cil.cil_target_build(dev(wl.target), dev(wl.target_normals))
    single = "point_to_point" if w[0] == 1.0 else "point_to_plane"
    a = cil.decode_result(cil.cil_icp_run(t, dev(wl.source), dev(np.eye(4)),
                                          cil.make_params("combined", 10, 1.0, w_point=w[0], w_plane=w[1]))[0])
    b = cil.decode_result(cil.cil_icp_run(t, dev(wl.source), dev(np.eye(4)), cil.make_params(single, 10, 1.0))[0])
    assert W.rot_angle(a.pose[:3, :3] @ b.pose[:3, :3].T) < 1e-9 and np.abs(a.pose[:3, 3] - b.pose[:3, 3]).max() < 1e-9
    assert a.n_corr == b.n_corr


def test_run_c3(cil):
    check_run(cil, W.c3(), "point_to_plane")


# ------------------------------------------------------------------ statuses and edge cases
def test_status_degenerate_no_corr_and_alias(cil):
    rng = np.random.default_rng(4)
    pts = rng.uniform(-1, 1, (500, 3)).astype(np.float32)
    pts[:, 2] = 0
    nrm = np.tile(np.array([[0, 0, 1]], np.float32), (500, 1))
    t = cil.cil_target_build(dev(pts), dev(nrm))
    prm = cil.make_params("point_to_plane", 5, 0.1)
    res_t, _ = cil.cil_icp_run(t, dev(pts + np.float32(0.01)), dev(np.eye(4)), prm)
    res = cil.decode_result(res_t)
    assert res.status == cil.CIL_ERR_DEGENERATE and not res.converged and res.iterations == 1
    assert np.array_equal(res.pose, np.eye(4))
    res_t, _ = cil.cil_icp_run(t, dev(pts + np.float32(100)), dev(np.eye(4)), prm)
    res = cil.decode_result(res_t)
    assert res.status == cil.CIL_NO_CORRESPONDENCES and res.n_corr == 0 and res.iterations == 1
    # in-place iterate (pose_in aliases pose_out), m == 0 -> no correspondences, pose kept
    P = dev(np.eye(4))
    P2, sys_t, _, _ = cil.cil_icp_iterate(t, torch.empty((0, 3), device="cuda"), P, prm, pose_out=P)
    assert cil.decode_system(sys_t).status == cil.CIL_NO_CORRESPONDENCES
    assert np.array_equal(P.cpu().numpy(), np.eye(4))
    # point-to-plane without normals is a host-side error
    t2 = cil.cil_target_build(dev(pts), None)
    with pytest.raises(cil.CilError) as e:
        cil.cil_icp_iterate(t2, dev(pts), P, prm)
    assert e.value.status == cil.CIL_ERR_NO_NORMALS


def test_converges_and_stops(cil):
    """tgt = src with tolerances -> converged after 1 iteration; later launches do nothing."""
    w = W.c4("point_to_plane", rings=8, az=4000)
    t = cil.cil_target_build(dev(w.target), dev(w.target_normals))
    prm = cil.make_params("point_to_plane", 20, 1.0, rot_tol=1e-5, trans_tol=1e-6)
    res_t, log = cil.cil_icp_run(t, dev(w.target), dev(np.eye(4)), prm)
    res = cil.decode_result(res_t)
    assert res.converged and res.iterations == 1 and res.rmse == 0.0 and res.n_corr == w.n
    assert (log.cpu().numpy()[1:] == 0).all()


def test_deterministic(cil):
    w = W.c4("point_to_plane", rings=16, az=8000)
    t = cil.cil_target_build(dev(w.target), dev(w.target_normals))
    prm = cil.make_params("point_to_plane", 10, 1.0)
    a = cil.decode_result(cil.cil_icp_run(t, dev(w.source), dev(np.eye(4)), prm)[0])
    b = cil.decode_result(cil.cil_icp_run(t, dev(w.source), dev(np.eye(4)), prm)[0])
    assert np.array_equal(a.pose, b.pose) and a.rmse == b.rmse


def test_icp_align_host_api(cil):
    """the e2e public call from host arrays"""
    w = W.c1()
    res = cil.icp_align(w.target, w.target_normals, w.source, "point_to_plane", 20, 0.1)
    o = oracle.icp_run(w.target, w.target_normals, w.source, "point_to_plane", 20, 0.1)
    assert W.rot_angle(res.pose[:3, :3] @ o.pose[:3, :3].T) <= 1e-4
    assert np.abs(res.pose[:3, 3] - o.pose[:3, 3]).max() <= 1e-5


# ------------------------------------------------------------------ NEXT-3: PCA normals
def _check_normals(cil, pts, k, view, min_gap=1e-3):
    """cil_estimate_normals vs oracle.pca_normals: where the k-NN set is unambiguous (the k-th
    and (k+1)-th fp64 distances differ by > 1e-6 relative) and the smallest eigenvalue is
    separated (relative eigengap > min_gap), the normals agree to 1e-6 rad and the curvature to
    1e-5 relative; wherever the k-NN set is unambiguous the normal's Rayleigh quotient equals the
    smallest eigenvalue and the curvature agrees; everywhere the GPU normal is a unit vector
    facing the viewpoint."""
    t = cil.cil_target_build(dev(pts), None)
    g, gc = cil.cil_estimate_normals(t, k, view, want_curvature=True)
    g, gc = g.cpu().numpy().astype(np.float64), gc.cpu().numpy().astype(np.float64)
    o, oc = oracle.pca_normals(pts, k, view=view)
    o = o.astype(np.float64)
    tree = oracle.KDTree(pts)
    idx, d2 = oracle.knn(None, pts.astype(np.float64), k=k + 1, tree=tree)
    clear = (d2[:, k] - d2[:, k - 1]) > 1e-6 * np.maximum(d2[:, k - 1], 1e-300)
    P = pts.astype(np.float64)[idx[:, :k]]
    Cv = np.einsum("nki,nkj->nij", P - P.mean(1, keepdims=True), P - P.mean(1, keepdims=True)) / k
    ev = np.linalg.eigvalsh(Cv)
    sep = (ev[:, 1] - ev[:, 0]) > min_gap * np.maximum(ev[:, 2], 1e-300)
    ok = clear & sep
    assert ok.mean() > 0.9, ok.mean()
    # angle from the cross product (arccos of a dot product near 1 is dominated by the fp32
    # rounding of the normals' lengths); both normals renormalised in fp64
    gn = g[ok] / np.linalg.norm(g[ok], axis=1, keepdims=True)
    on = o[ok] / np.linalg.norm(o[ok], axis=1, keepdims=True)
    ang = np.arcsin(np.clip(np.linalg.norm(np.cross(gn, on), axis=1), 0, 1))
    assert ang.max() <= 1e-6, ang.max()
    assert ((g[ok] * o[ok]).sum(1) > 0).all()                     # same orientation
    np.testing.assert_allclose(gc[ok], oc[ok].astype(np.float64), rtol=1e-5, atol=1e-9)
    # every point with an unambiguous k-NN set, whatever its eigengap: the direction is
    # ill-conditioned where the two smallest eigenvalues meet, but the Rayleigh quotient of the
    # GPU normal on the oracle-side covariance is not -- it must sit at the smallest eigenvalue
    # (within 1e-5 of the spectrum's scale), and so must the curvature
    gu = g[clear] / np.linalg.norm(g[clear], axis=1, keepdims=True)
    ray = np.einsum("ni,nij,nj->n", gu, Cv[clear], gu)
    assert (ray <= ev[clear, 0] + 1e-5 * np.maximum(ev[clear, 2], 1e-300)).all(), \
        float((ray - ev[clear, 0]).max())
    np.testing.assert_allclose(gc[clear], oc[clear].astype(np.float64), rtol=1e-5, atol=1e-9)
    np.testing.assert_allclose(np.linalg.norm(g, axis=1), 1.0, atol=1e-6)
    assert (((np.asarray(view) - pts.astype(np.float64)) * g).sum(1) >= -1e-6).all()
    return ok.mean()


@pytest.mark.parametrize("n,k", [(3000, 10), (20000, 6), (5000, 16)])
def test_normals_random_surface(cil, n, k):
    rng = np.random.default_rng(n + k)
    u, v = rng.uniform(-1, 1, (2, n))
    pts = np.stack([u, v, 0.2 * np.sin(2 * u) * np.cos(v)], 1) + rng.normal(0, 0.002, (n, 3))
    _check_normals(cil, pts.astype(np.float32), k, (0.3, -0.2, 5.0))


def test_normals_c3_config(cil):
    """BASELINE.json configs[2]: the 640x480 depth frame, 10-NN, viewpoint at the camera."""
    w = gen.c3_depth()
    frac = _check_normals(cil, w.target, 10, (0.0, 0.0, 0.0))
    assert frac > 0.95


@pytest.mark.parametrize("pinned", [True, False])
@pytest.mark.parametrize("metric", ["point_to_plane", "point_to_point"])
def test_align_host_equals_device_path(cil, metric, pinned):
    """cil_icp_align_host (HOST buffers in, result out, one C call) = cil_target_build +
    cil_icp_run on device buffers, bit for bit; pinned and pageable inputs; a given initial pose
    and the NULL (identity) one; against the oracle within the north_star tolerances"""
    w = W.c4(metric, 16, 8000)
    prm = cil.make_params(metric, 12, w.max_dist)
    t = cil.cil_target_build(dev(w.target), dev(w.target_normals))
    hold = (lambda a: torch.as_tensor(np.ascontiguousarray(a)).pin_memory()) if pinned else \
        (lambda a: torch.as_tensor(np.ascontiguousarray(a)))
    for P0 in (None, w.gt_pose @ np.array([[1, 0, 0, 0.05], [0, 1, 0, -0.02], [0, 0, 1, 0.01], [0, 0, 0, 1.0]])):
        d_p0 = dev(np.eye(4) if P0 is None else P0)
        ref = cil.decode_result(cil.cil_icp_run(t, dev(w.source), d_p0, prm, want_log=False)[0])
        got = cil.cil_icp_align_host(hold(w.target), hold(w.target_normals), hold(w.source), P0, prm)
        assert got.status == ref.status == 0 and got.iterations == ref.iterations == 12
        assert got.n_corr == ref.n_corr and got.rmse == ref.rmse
        assert np.array_equal(got.pose, ref.pose)
    o = oracle.icp_run(w.target, w.target_normals, w.source, metric, 12, w.max_dist)
    got = cil.cil_icp_align_host(hold(w.target), hold(w.target_normals), hold(w.source), None, prm)
    assert W.rot_angle(got.pose[:3, :3] @ o.pose[:3, :3].T) <= 1e-4
    assert np.abs(got.pose[:3, 3] - o.pose[:3, 3]).max() <= 1e-5
    t.free()


def test_align_host_errors_and_edge_cases(cil):
    """missing normals for point-to-plane -> CIL_ERR_NO_NORMALS (nothing leaks: the call can be
    repeated); an empty source -> CIL_NO_CORRESPONDENCES on the device, identity pose; the small
    brute-force path (C1) through the host call"""
    w = W.c1()
    prm = cil.make_params("point_to_plane", 5, w.max_dist)
    for _ in range(3):
        with pytest.raises(cil.CilError) as ei:
            cil.cil_icp_align_host(w.target, None, w.source, None, prm)
        assert ei.value.status == cil.CIL_ERR_NO_NORMALS
    r = cil.cil_icp_align_host(w.target, w.target_normals, np.zeros((0, 3), np.float32), None, prm)
    assert r.status == cil.CIL_NO_CORRESPONDENCES and np.array_equal(r.pose, np.eye(4))
    t = cil.cil_target_build(dev(w.target), dev(w.target_normals))
    ref = cil.decode_result(cil.cil_icp_run(t, dev(w.source), dev(np.eye(4)), prm, want_log=False)[0])
    got = cil.cil_icp_align_host(w.target, w.target_normals, w.source, None, prm)
    assert got.status == 0 and np.array_equal(got.pose, ref.pose) and got.n_corr == ref.n_corr
    t.free()


def test_run_empty_source(cil):
    """cil_icp_run with m = 0: CIL_NO_CORRESPONDENCES after one iteration, identity pose"""
    w = W.c1()
    t = cil.cil_target_build(dev(w.target), dev(w.target_normals))
    empty = torch.empty((0, 3), dtype=torch.float32, device="cuda")
    res = cil.decode_result(cil.cil_icp_run(t, empty, dev(np.eye(4)), cil.make_params("point_to_plane", 5, 0.1))[0])
    assert res.status == cil.CIL_NO_CORRESPONDENCES and res.iterations == 1 and np.array_equal(res.pose, np.eye(4))


def test_normals_non_finite_point(cil):
    """a NaN target point must not fault the normal kernel: it gets a zero normal, the others
    are unit vectors (cil.h: fewer than 3 finite neighbours -> zero normal)"""
    rng = np.random.default_rng(5)
    P = np.stack([rng.random(3000), rng.random(3000), np.zeros(3000)], 1).astype(np.float32)
    P[17] = np.nan
    t = cil.cil_target_build(dev(P), None)
    n, c = cil.cil_estimate_normals(t, 10, (0.0, 0.0, 1.0))
    n = n.cpu().numpy()
    assert np.array_equal(n[17], np.zeros(3, np.float32))
    ok = np.ones(3000, bool); ok[17] = False
    assert np.allclose(np.linalg.norm(n[ok], axis=1), 1.0, atol=1e-5)
