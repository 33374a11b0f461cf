"""GPU parity of the leaf-neighbour-list search (csrc/lnl.cu): the per-query list
scan returns exactly what the packet engine returns (the exact minimum of the same fp32 d2 with the
lowest-index tie rule), so every result with the lists must equal the result without them BIT FOR BIT,
and both must match the fp64 oracle within the north_star tolerances."""
import numpy as np
import pytest
import torch

import oracle
from tests import workloads as W
from tests.test_gpu_parity import check_nn, dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cil():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1807_00399_b200 as cil
    return cil


def _clouds(kind, rng):
    n, m = 20000, 30000
    if kind == "uniform":
        T = rng.random((n, 3))
        Q = rng.random((m, 3))
    elif kind == "dups":          # heavy exact duplicates: zero box distances, ties everywhere
        T = np.repeat(rng.random((n // 50, 3)), 50, 0)
        Q = T[rng.integers(0, T.shape[0], m)] + rng.normal(0, 1e-3, (m, 3)) * (rng.random((m, 1)) < 0.5)
    elif kind == "line":
        T = np.stack([rng.random(n), np.zeros(n), np.zeros(n)], 1)
        Q = rng.random((m, 3)) * [1.0, 0.01, 0.01]
    elif kind == "far":
        T = rng.random((n, 3))
        Q = rng.standard_normal((m, 3)) * 20.0
    else:                          # log-radial, strongly non-uniform
        r = np.exp(rng.uniform(0, 5, n))
        a = rng.uniform(0, 2 * np.pi, n)
        T = np.stack([r * np.cos(a), r * np.sin(a), rng.normal(0, 0.01, n)], 1)
        Q = T[rng.integers(0, n, m)] + rng.normal(0, 0.05, (m, 3))
    return T.astype(np.float32), Q.astype(np.float32)


@pytest.mark.parametrize("kind", ["uniform", "dups", "line", "far", "radial"])
@pytest.mark.parametrize("leaf_size,lists", [(16, 0), (4, 1), (8, 16), (32, 256)])
def test_nn_lists_equal_engine(cil, kind, leaf_size, lists):
    rng = np.random.default_rng(hash((kind, leaf_size, lists)) % 2**32)
    T, Q = _clouds(kind, rng)
    res = []
    for ll in (lists, -1):
        t = cil.cil_target_build(dev(T), None, leaf_size=leaf_size, leaf_lists=ll)
        gi, gd = cil.cil_nn_query(t, dev(Q))
        res.append((gi.cpu().numpy(), gd.cpu().numpy()))
        t.free()
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1].view(np.uint32), res[1][1].view(np.uint32))
    o_idx, o_d2 = oracle.knn(T, Q.astype(np.float64), k=2)
    check_nn(T, Q.astype(np.float64), res[0][0], res[0][1], o_idx, o_d2)


@pytest.mark.parametrize("pose", ["identity", "gt"])
def test_iterate_c4_lists_equal_engine(cil, pose):
    """Full-size C4 stateless iterate: correspondences and d2 with the lists == without, bitwise."""
    w = W.c4("point_to_plane")
    P = np.eye(4) if pose == "identity" else w.gt_pose
    out = []
    for ll in (0, -1):
        t = cil.cil_target_build(dev(w.target), dev(w.target_normals), leaf_lists=ll)
        prm = cil.make_params("point_to_plane", 1, w.max_dist)
        ws = cil.alloc_workspace(w.m, prm)
        r = cil.cil_icp_iterate(t, dev(w.source), dev(P), prm, ws=ws, want_corr=True)
        out.append([x.cpu().numpy() if torch.is_tensor(x) else x for x in r])
        t.free()
    ia, da = out[0][-2], out[0][-1]
    ib, db = out[1][-2], out[1][-1]
    assert np.array_equal(ia, ib)
    assert np.array_equal(np.asarray(da).view(np.uint32), np.asarray(db).view(np.uint32))


@pytest.mark.parametrize("metric", ["point_to_plane", "point_to_point"])
def test_run_c4_lists_equal_engine(cil, metric):
    """Full-size C4 certified 50-iteration run: the pose with the lists is bitwise the pose without
    them (every iteration's correspondences are the exact NN either way)."""
    w = W.c4(metric)
    poses = []
    for ll in (0, -1):
        t = cil.cil_target_build(dev(w.target), dev(w.target_normals), leaf_lists=ll)
        prm = cil.make_params(metric, w.max_iters, w.max_dist)
        res_t, _ = cil.cil_icp_run(t, dev(w.source), dev(np.eye(4)), prm)
        poses.append(cil.decode_result(res_t))
        t.free()
    assert np.array_equal(poses[0].pose, poses[1].pose)
    assert poses[0].n_corr == poses[1].n_corr and poses[0].status == poses[1].status
