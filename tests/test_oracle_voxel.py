"""Pins for the voxel-grid downsampling oracle (oracle.voxel_downsample; SURVEY.md 8(f) NEXT-4,
PAPER.md:125, R27-R29) against things other than
itself: SPEC's worked two-bin example, the single-bin case, a brute-force hash grouping written
here with numpy + a Python dict, and the invariants SPEC states (count <= n, each output inside
its bin's half-open cube, idempotence on bin keys).  CPU only.
"""
import math

import numpy as np
import pytest

import gen
import oracle


def test_spec_two_bin_example():
    """x in {0.1, 0.2, 0.9}, bin 0.5 -> 0.15 (bin 0) and 0.9 (bin 1)"""
    p = np.array([[0.1, 0, 0], [0.2, 0, 0], [0.9, 0, 0]], np.float32)
    out, _, keys = oracle.voxel_downsample(p, 0.5)
    np.testing.assert_array_equal(keys, [[0, 0, 0], [1, 0, 0]])
    assert out[0, 0] == np.float32((np.float64(np.float32(0.1)) + np.float64(np.float32(0.2))) / 2)
    assert out[1, 0] == np.float32(0.9)


def test_single_bin_is_the_centroid():
    rng = np.random.default_rng(3)
    p = (rng.random((1000, 3)) * 0.99).astype(np.float32)
    out, _, keys = oracle.voxel_downsample(p, 1.0)
    assert out.shape == (1, 3) and keys.tolist() == [[0, 0, 0]]
    np.testing.assert_allclose(out[0], p.astype(np.float64).mean(0), rtol=1e-7)


def _brute(p, h, origin, nrm=None):
    """hash-group brute force: dict key -> list of indices, in input order"""
    groups = {}
    P = p.astype(np.float64)
    for i in range(p.shape[0]):
        k = tuple(int(math.floor((P[i, a] - origin[a]) / h)) for a in range(3))
        groups.setdefault(k, []).append(i)
    keys = sorted(groups)
    pts = np.array([P[groups[k]].mean(0) for k in keys])
    out_n = None
    if nrm is not None:
        N = nrm.astype(np.float64)
        ms = [N[groups[k]].mean(0) for k in keys]
        out_n = np.array([m / np.linalg.norm(m) if np.linalg.norm(m) >= 1e-12 else np.zeros(3) for m in ms])
    return np.array(keys, np.int64), pts, out_n


@pytest.mark.parametrize("h,origin", [(0.05, (0.0, 0.0, 0.0)), (0.013, (0.3, -0.2, 0.01))])
def test_matches_hash_group_brute_force(h, origin):
    """10^4 random points -> identical keys, centroids within 1e-12 (fp64 means
    before the fp32 cast, here compared after it: within 1 fp32 ulp)"""
    rng = np.random.default_rng(11)
    p = (rng.random((10000, 3)) * 2.0 - 0.5).astype(np.float32)
    nrm = rng.standard_normal((10000, 3)).astype(np.float32)
    out, on, keys = oracle.voxel_downsample(p, h, origin, normals=nrm)
    bk, bp, bn = _brute(p, h, origin, nrm)
    np.testing.assert_array_equal(keys, bk)
    np.testing.assert_allclose(out, bp, rtol=2 ** -23, atol=1e-12)
    np.testing.assert_allclose(on, bn, rtol=1e-6, atol=1e-6)


def test_invariants_containment_idempotence():
    """count <= n; every output lies in its bin's half-open cube (up to the
    fp32 rounding of the mean); downsampling the output again keeps every bin key"""
    w = gen.c3_depth()
    h = 0.01
    out, _, keys = oracle.voxel_downsample(w.target, h)
    assert 0 < out.shape[0] <= w.n
    lo = keys * h
    o64 = out.astype(np.float64)
    eps = 1e-6
    assert np.all(o64 >= lo - eps) and np.all(o64 < lo + h + eps)
    out2, _, keys2 = oracle.voxel_downsample(out, h)
    # points that rounded onto a bin face may move by one bin; all others keep their key
    inside = np.all((o64 > lo + eps) & (o64 < lo + h - eps), 1)
    k2 = {tuple(k) for k in keys2}
    assert all(tuple(k) in k2 for k in keys[inside])
    assert out2.shape[0] <= out.shape[0]


def test_zero_mean_normal_and_key_range():
    p = np.array([[0.1, 0.1, 0.1], [0.2, 0.2, 0.2], [5.0, 5.0, 5.0]], np.float32)
    nrm = np.array([[0, 0, 1], [0, 0, -1], [0, 1, 0]], np.float32)
    out, on, keys = oracle.voxel_downsample(p, 1.0, normals=nrm)
    np.testing.assert_array_equal(on, [[0, 0, 0], [0, 1, 0]])     # opposite normals cancel -> 0
    np.testing.assert_array_equal(keys, [[0, 0, 0], [5, 5, 5]])
    with pytest.raises(ValueError):
        oracle.voxel_downsample(np.array([[1e30, 0, 0]], np.float32), 1e-3)
    neg, _, kn = oracle.voxel_downsample(np.array([[-0.5, -1e-9, 0.0]], np.float32), 1.0)
    np.testing.assert_array_equal(kn, [[-1, -1, 0]])                # floor, not truncation
