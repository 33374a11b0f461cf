"""CPU-side checks of the C ABI boundary (no GPU needed): libcil.so loads, exports every
function include/cil.h declares, the ctypes struct layouts equal the C layouts, and the
host-detectable argument errors are returned before anything touches the device."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "cil.h")


def _declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cil_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def cil():
    import paper_1807_00399_b200 as cil
    return cil


def test_library_exports_every_declared_symbol(cil):
    names = _declared_functions()
    assert len(names) >= 10
    for n in names:
        assert hasattr(cil.lib(), n), f"libcil.so does not export {n}"
    assert sorted(cil.EXPORTED) == names
    assert "sm_100a" in cil.version()


def test_struct_layouts_match_header(cil):
    """Compile a probe against include/cil.h and compare sizeof/offsetof with ctypes."""
    probe = r"""
#include <stdio.h>
#include <stddef.h>
#include "cil.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu\n", sizeof(cil_index_params), sizeof(cil_icp_params), sizeof(cil_icp_result),
         sizeof(cil_icp_system), sizeof(cil_target_info), sizeof(cil_intrinsics));
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\n", offsetof(cil_icp_params, max_corr_dist), offsetof(cil_icp_result, rmse),
         offsetof(cil_icp_result, status), offsetof(cil_icp_system, sse), offsetof(cil_icp_system, status),
         offsetof(cil_target_info, device_bytes), offsetof(cil_intrinsics, fx), offsetof(cil_intrinsics, cy),
         offsetof(cil_index_params, index_kind), offsetof(cil_index_params, grid_points), offsetof(cil_target_info, index_kind));
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "p.c")
        exe = os.path.join(d, "p")
        open(c, "w").write(probe)
        subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        out = subprocess.check_output([exe]).decode().split()
    sizes = [int(x) for x in out[:6]]
    offs = [int(x) for x in out[6:]]
    assert sizes == [C.sizeof(cil.cil_index_params), C.sizeof(cil.cil_icp_params), C.sizeof(cil.cil_icp_result),
                     C.sizeof(cil.cil_icp_system), C.sizeof(cil.cil_target_info), C.sizeof(cil.cil_intrinsics)]
    assert offs == [cil.cil_icp_params.max_corr_dist.offset, cil.cil_icp_result.rmse.offset,
                    cil.cil_icp_result.status.offset, cil.cil_icp_system.sse.offset,
                    cil.cil_icp_system.status.offset, cil.cil_target_info.device_bytes.offset,
                    cil.cil_intrinsics.fx.offset, cil.cil_intrinsics.cy.offset,
                    cil.cil_index_params.index_kind.offset, cil.cil_index_params.grid_points.offset,
                    cil.cil_target_info.index_kind.offset]


def test_host_side_argument_errors(cil):
    L = cil.lib()
    h = C.c_void_p()
    assert L.cil_target_build(None, None, 0, None, None, C.byref(h)) == cil.CIL_ERR_EMPTY_TARGET
    assert L.cil_target_build(None, None, -5, None, None, C.byref(h)) == cil.CIL_ERR_INVALID_ARG
    assert L.cil_target_build(None, None, 10, None, None, C.byref(h)) == cil.CIL_ERR_INVALID_ARG
    assert L.cil_target_build(None, None, 2 ** 31, None, None, C.byref(h)) == cil.CIL_ERR_INVALID_ARG
    assert L.cil_target_build(None, None, 10, None, None, None) == cil.CIL_ERR_INVALID_ARG
    bad = cil.cil_index_params()
    bad.leaf_size = 7
    assert L.cil_target_build(C.c_void_p(256), None, 10, C.byref(bad), None, C.byref(h)) == cil.CIL_ERR_INVALID_ARG
    assert "leaf_size" in L.cil_last_error().decode()
    bad = cil.cil_index_params()
    bad.index_kind = 7
    assert L.cil_target_build(C.c_void_p(256), None, 10, C.byref(bad), None, C.byref(h)) == cil.CIL_ERR_INVALID_ARG
    assert "index_kind" in L.cil_last_error().decode()
    bad = cil.cil_index_params()
    bad.index_kind = cil.CIL_INDEX_GRID
    for gp in (-1.0, float("nan"), float("inf")):
        bad.grid_points = gp
        assert L.cil_target_build(C.c_void_p(256), None, 10, C.byref(bad), None, C.byref(h)) == cil.CIL_ERR_INVALID_ARG
        assert "grid_points" in L.cil_last_error().decode()
    assert L.cil_nn_query(None, None, 10, 1.0, None, None, None) == cil.CIL_ERR_INVALID_ARG
    p = cil.make_params("point_to_plane", 10, 0.1)
    assert L.cil_icp_iterate(None, None, 10, None, C.byref(p), None, 0, None, None, None, None, None) == \
        cil.CIL_ERR_INVALID_ARG
    assert L.cil_icp_run(None, None, 10, None, C.byref(p), None, 0, None, None, None) == cil.CIL_ERR_INVALID_ARG
    # the host-buffer call: argument errors come back before any CUDA call
    r = cil.cil_icp_result()
    hp = C.c_void_p(4096)
    assert L.cil_icp_align_host(hp, None, 10, hp, 10, None, C.byref(p), None, None, None) == cil.CIL_ERR_INVALID_ARG
    assert L.cil_icp_align_host(hp, None, 10, hp, 10, None, None, None, C.byref(r), None) == cil.CIL_ERR_INVALID_ARG
    assert L.cil_icp_align_host(hp, None, 0, hp, 10, None, C.byref(p), None, C.byref(r), None) == cil.CIL_ERR_EMPTY_TARGET
    assert L.cil_icp_align_host(hp, None, -1, hp, 10, None, C.byref(p), None, C.byref(r), None) == cil.CIL_ERR_INVALID_ARG
    assert L.cil_icp_align_host(hp, None, 10, hp, 2 ** 31, None, C.byref(p), None, C.byref(r), None) == cil.CIL_ERR_INVALID_ARG
    assert L.cil_icp_align_host(None, None, 10, hp, 10, None, C.byref(p), None, C.byref(r), None) == cil.CIL_ERR_INVALID_ARG
    assert L.cil_icp_align_host(hp, None, 10, None, 10, None, C.byref(p), None, C.byref(r), None) == cil.CIL_ERR_INVALID_ARG
    assert L.cil_target_free(None, None) == cil.CIL_OK
    assert L.cil_status_string(cil.CIL_ERR_DEGENERATE) == b"CIL_ERR_DEGENERATE"


def test_workspace_bytes_host_only(cil):
    p = cil.make_params("point_to_plane", 50, 1.0)
    a = cil.cil_icp_workspace_bytes(1000, p)
    b = cil.cil_icp_workspace_bytes(2_000_000, p)
    assert a > 0 and b > a and a % 256 == 0 and b % 256 == 0
    assert b - a >= 4 * (2_000_000 - 1000) - 256     # per-point warm-start state
    assert cil.cil_icp_workspace_bytes(-1, p) == 0
    assert cil.cil_icp_workspace_bytes(2 ** 31, p) == 0


def test_no_oracle_in_product_path():
    """The product package never imports or links the oracle (boundary)."""
    pkg = os.path.join(ROOT, "paper_1807_00399_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "liboracle" not in txt and "orc_" not in txt, f


def test_combined_metric_parameter_errors(cil):
    """CIL_COMBINED: weights finite, >= 0, not both 0; the single
    metrics keep w_point = w_plane = 0.  Rejected on the host, before the target is touched."""
    L = cil.lib()
    for wp, wl in ((0.0, 0.0), (-1.0, 1.0), (1.0, float("nan")), (float("inf"), 1.0)):
        p = cil.make_params("combined", 5, 0.1, w_point=wp, w_plane=wl)
        assert L.cil_icp_run(None, None, 10, None, C.byref(p), None, 0, None, None, None) == cil.CIL_ERR_INVALID_ARG
        assert "weights" in L.cil_last_error().decode()
    p = cil.make_params("point_to_plane", 5, 0.1, w_point=1.0)
    assert L.cil_icp_iterate(None, None, 10, None, C.byref(p), None, 0, None, None, None, None, None) == \
        cil.CIL_ERR_INVALID_ARG
    assert "CIL_COMBINED" in L.cil_last_error().decode()
    ok = cil.make_params("combined", 5, 0.1, w_point=0.5, w_plane=1.0)
    assert L.cil_icp_run(None, None, 10, None, C.byref(ok), None, 0, None, None, None) == cil.CIL_ERR_INVALID_ARG
    assert "target" in L.cil_last_error().decode()        # parameters passed; the NULL target is next


def test_projective_argument_errors(cil):
    """cil_proj_* (SURVEY.md 8(f) NEXT-2): intrinsics, normals and workspace are validated on
    the host; the workspace is O(1) in m."""
    L = cil.lib()
    p = cil.make_params("point_to_plane", 5, 0.05)
    K = cil.make_intrinsics(640, 480, 525.0, 525.0, 319.5, 239.5)
    nb = cil.cil_proj_workspace_bytes(1000, p)
    assert nb > 0 and nb % 256 == 0 and nb == cil.cil_proj_workspace_bytes(2_000_000, p)
    assert cil.cil_proj_workspace_bytes(-1, p) == 0
    fake = C.c_void_p(1 << 20)
    ws = C.c_void_p(1 << 24)
    args = lambda K_, nrm, m=10: (fake, nrm, C.byref(K_) if K_ is not None else None, fake, m, fake, C.byref(p), ws,
                                  nb, fake, None, None, None, None)
    assert L.cil_proj_iterate(*args(None, fake)) == cil.CIL_ERR_INVALID_ARG
    for bad in (cil.make_intrinsics(0, 480, 525, 525, 1, 1), cil.make_intrinsics(640, 480, 0.0, 525, 1, 1),
                cil.make_intrinsics(640, 480, 525, float("nan"), 1, 1), cil.make_intrinsics(1 << 16, 1 << 16, 1, 1, 0, 0)):
        assert L.cil_proj_iterate(*args(bad, fake)) == cil.CIL_ERR_INVALID_ARG
    assert L.cil_proj_iterate(*args(K, None)) == cil.CIL_ERR_NO_NORMALS
    assert L.cil_proj_iterate(*args(K, fake, m=-1)) == cil.CIL_ERR_INVALID_ARG
    a = list(args(K, fake)); a[8] = nb - 256
    assert L.cil_proj_iterate(*a) == cil.CIL_ERR_WORKSPACE
    p0 = cil.make_params("point_to_plane", 0, 0.05)
    assert L.cil_proj_run(fake, fake, C.byref(K), fake, 10, fake, C.byref(p0), ws, nb, fake, None, None) == \
        cil.CIL_ERR_INVALID_ARG


def test_voxel_argument_errors(cil):
    """cil_voxel_downsample: host-side validation"""
    L = cil.lib()
    fake = C.c_void_p(1 << 20)
    o = (C.c_double * 3)(0.0, 0.0, 0.0)
    assert L.cil_voxel_downsample(fake, None, -1, 0.01, C.byref(o), fake, None, fake, None) == cil.CIL_ERR_INVALID_ARG
    for b in (0.0, -1.0, float("nan"), float("inf")):
        assert L.cil_voxel_downsample(fake, None, 10, b, C.byref(o), fake, None, fake, None) == cil.CIL_ERR_INVALID_ARG
    bad = (C.c_double * 3)(0.0, float("nan"), 0.0)
    assert L.cil_voxel_downsample(fake, None, 10, 0.01, C.byref(bad), fake, None, fake, None) == cil.CIL_ERR_INVALID_ARG
    assert L.cil_voxel_downsample(fake, None, 10, 0.01, None, fake, None, None, None) == cil.CIL_ERR_INVALID_ARG
    assert L.cil_voxel_downsample(None, None, 10, 0.01, None, fake, None, fake, None) == cil.CIL_ERR_INVALID_ARG
    assert L.cil_voxel_downsample(fake, None, 10, 0.01, None, fake, fake, fake, None) == cil.CIL_ERR_NO_NORMALS


def test_engine_trace_needs_a_trace_build(cil):
    """The default build compiles the diagnostic engine trace out (include/cil.h): a non-NULL
    buffer is refused with CIL_ERR_INVALID_ARG and a message; NULL (off) is accepted."""
    buf = (C.c_int32 * 64)()
    rc = cil.lib().cil_debug_engine_trace(C.cast(buf, C.c_void_p))
    assert rc == cil.CIL_ERR_INVALID_ARG
    assert b"CIL_TRACE" in cil.lib().cil_last_error()
    assert cil.lib().cil_debug_engine_trace(None) == cil.CIL_OK
