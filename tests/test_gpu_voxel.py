"""GPU parity of voxel-grid downsampling (cil_voxel_downsample, DESIGN.md
R27-R29) against the fp64 oracle (oracle.voxel_downsample) on the same seeded inputs, through
the C ABI.  Both sides compute the keys with the same correctly rounded fp64 operations and sum
each bin in increasing input index, so the bin count, the order and every output float are
compared bit for bit.
"""
import numpy as np
import pytest
import torch

import gen
import oracle
from tests import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cil():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1807_00399_b200 as cil
    return cil


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a)).cuda()


def check(cil, pts, h, origin=(0.0, 0.0, 0.0), nrm=None):
    op, on, ok = oracle.voxel_downsample(pts, h, origin, normals=nrm)
    gp, gn = cil.cil_voxel_downsample(dev(pts), h, origin, normals=dev(nrm) if nrm is not None else None)
    gp = gp.cpu().numpy()
    assert gp.shape == op.shape
    np.testing.assert_array_equal(gp, op)
    if nrm is not None:
        np.testing.assert_array_equal(gn.cpu().numpy(), on)
    return op.shape[0]


@pytest.mark.parametrize("n,h", [(1, 0.1), (7, 0.5), (4095, 0.05), (4097, 0.05), (10000, 0.05), (100003, 0.02)])
def test_voxel_random_ragged(cil, n, h):
    rng = np.random.default_rng(n)
    p = (rng.random((n, 3)) * 2.0 - 1.0).astype(np.float32)
    nrm = rng.standard_normal((n, 3)).astype(np.float32)
    check(cil, p, h, (0.013, -0.2, 0.3), nrm)


@pytest.mark.parametrize("n", [255, 257, 2049, 8193, 16384, 16385, 32769, 65537, 131073, 262145, 300001])
def test_voxel_sort_tile_regimes(cil, n):
    """sizes on both sides of every sort-tile size (256 ... 4096 keys per CTA, up to 64 CTAs per
    pass for small inputs) and of the one-block / three-kernel scan of the digit x tile table:
    the stable radix sort decides the bins' input order, so the means are bit-exact only if it
    is right"""
    rng = np.random.default_rng(n)
    p = (rng.random((n, 3)) * 4.0 - 2.0).astype(np.float32)
    check(cil, p, 0.03, (0.0, 0.1, -0.2))


def test_voxel_c3_one_centimetre(cil):
    """the paper's ICP preprocessing: 1 cm voxels on the C3 depth frame"""
    w = W.c3()
    nb = check(cil, w.target, 0.01, nrm=w.target_normals)
    assert 1000 < nb < w.n


def test_voxel_c4_lidar(cil):
    w = W.c4("point_to_plane", rings=16, az=8000)
    check(cil, w.target, 0.05, nrm=w.target_normals)
    check(cil, w.target, 0.2)


def test_voxel_single_bin_duplicates_and_negative(cil):
    p = np.full((3000, 3), 0.25, np.float32)
    assert check(cil, p, 1.0) == 1
    q = np.array([[-0.5, -1e-9, 0.0], [-1.0, -1.0, -1.0], [-1.0, -1.0, -1.0], [0.999, 0.0, -0.001]], np.float32)
    check(cil, q, 1.0)


def test_voxel_errors_on_device(cil):
    """a key outside int32 / non-finite coordinates / a span >= 2^21 bins -> *n_out = -1"""
    for p, h in ((np.array([[1e30, 0, 0]], np.float32), 1e-3),
                 (np.array([[0, 0, 0], [np.nan, 0, 0]], np.float32), 0.1),
                 (np.array([[0, 0, 0], [3000.0, 0, 0]], np.float32), 1e-3)):
        with pytest.raises(cil.CilError):
            cil.cil_voxel_downsample(dev(p), h)
    out, _ = cil.cil_voxel_downsample(torch.empty((0, 3), dtype=torch.float32, device="cuda"), 0.1)
    assert out.shape[0] == 0


def test_voxel_c4_full_size(cil):
    """the full 2 M-point C4 target (BASELINE.json configs[3]) at 5 cm, with normals: bit-exact"""
    w = W.c4("point_to_plane")
    nb = check(cil, w.target, 0.05, nrm=w.target_normals)
    assert 100_000 < nb < w.n
