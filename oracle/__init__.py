"""ctypes wrapper over liboracle.so -- the fp64 CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: import this from tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, nowhere else.  The product package
(paper_1807_00399_b200) never imports it.

Parity status of each function:
  knn / kd-tree ........... pinned (brute force, scipy cKDTree, self-query, ties)
  icp_system (H, g) ....... pinned (closed-form pairs, finite-difference Jacobian,
                             numpy dense J^T J, linearisation identity)
  solve_update ............ pinned (numpy.linalg.solve, scipy Rotation.from_rotvec)
  icp_run ................. pinned (Kabsch/SVD fixed point, planted-motion recovery,
                             translation-only closed form, equivariance)
  proj_system / proj_run .. pinned (identity self-pairing, one-pixel shift closed form,
                             half-away-from-zero rounding, bounds/invalid/rejection cases,
                             accumulation = icp_system_from_corr on the same pairs)
  voxel_downsample ........ pinned (SPEC two-bin example, single bin, numpy/dict hash-group
                             brute force, half-open cube containment, idempotence)
  pca_normals ............. pinned (noise-free planes, numpy eigh on explicit neighbourhoods)
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

OK, DEGENERATE, NO_CORRESPONDENCES = 0, 16, 17
METRICS = {"point_to_point": 0, "point_to_plane": 1, "combined": 2}

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


def _opt(t):
    """nullable ndpointer"""
    base = t

    class _Opt(base):  # type: ignore[misc, valid-type]
        @classmethod
        def from_param(cls, obj):
            if obj is None:
                return None
            return base.from_param(obj)
    return _Opt


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"oracle library missing: {_LIB_PATH} (run `make oracle` or __graft_entry__.build())")
        L = C.CDLL(_LIB_PATH)
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_get_threads.restype = C.c_int
        L.orc_kd_build.restype = C.c_void_p
        L.orc_kd_build.argtypes = [_f32p, C.c_int64, C.c_int]
        L.orc_kd_free.argtypes = [C.c_void_p]
        L.orc_knn.argtypes = [C.c_void_p, _f32p, C.c_int64, _f64p, C.c_int64, C.c_int, C.c_double, _i64p, _f64p]
        L.orc_transform.argtypes = [_f64p, _f32p, C.c_int64, _f64p]
        L.orc_set_combined_weights.argtypes = [C.c_double, C.c_double]
        L.orc_set_combined_weights.restype = None
        L.orc_icp_system.argtypes = [C.c_void_p, _f32p, _opt(_f32p), C.c_int64, _f32p, C.c_int64, _f64p, C.c_int,
                                     C.c_double, _f64p, _f64p, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                     _opt(_f64p), _opt(_f64p), _opt(_i64p), _opt(_f64p), _opt(_f64p)]
        L.orc_icp_system_from_corr.argtypes = [_f32p, _opt(_f32p), C.c_int64, _f32p, C.c_int64, _f64p, C.c_int, _i32p,
                                               _f64p, _f64p, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                               _opt(_f64p), _opt(_f64p)]
        L.orc_rodrigues.argtypes = [_f64p, _f64p]
        L.orc_solve_update.argtypes = [_f64p, _f64p, C.c_int64, _f64p, _f64p, _f64p,
                                       C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.orc_icp_run.argtypes = [C.c_void_p, _f32p, _opt(_f32p), C.c_int64, _f32p, C.c_int64, _f64p, C.c_int, C.c_int,
                                  C.c_double, C.c_double, C.c_double, _f64p, C.POINTER(C.c_double),
                                  C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                  C.POINTER(C.c_int32), _opt(_f64p), _opt(_f64p), _opt(_f64p), _opt(_f64p)]
        L.orc_proj_system.argtypes = [_f32p, _opt(_f32p), C.c_int64, C.c_int64, _f64p, _f32p, C.c_int64, _f64p,
                                      C.c_int, C.c_double, _f64p, _f64p, C.POINTER(C.c_double),
                                      C.POINTER(C.c_int64), _opt(_f64p), _opt(_f64p), _opt(_i64p), _opt(_f64p),
                                      _opt(_f64p)]
        L.orc_proj_run.argtypes = [_f32p, _opt(_f32p), C.c_int64, C.c_int64, _f64p, _f32p, C.c_int64, _f64p, C.c_int,
                                   C.c_int, C.c_double, C.c_double, C.c_double, _f64p, C.POINTER(C.c_double),
                                   C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                   C.POINTER(C.c_int32), _opt(_f64p), _opt(_f64p), _opt(_f64p), _opt(_f64p)]
        L.orc_voxel_downsample.restype = C.c_int64
        L.orc_voxel_downsample.argtypes = [_f32p, _opt(_f32p), C.c_int64, C.c_double, _f64p, _f32p, _opt(_f32p),
                                           _opt(_i64p)]
        L.orc_pca_normals.argtypes = [C.c_void_p, _f32p, C.c_int64, C.c_int, _f64p, _f32p, _opt(_f32p)]
        _lib = L
    return _lib


def set_combined_weights(w_point: float, w_plane: float) -> None:
    """weights of metric "combined" (w_point * point-to-point + w_plane * point-to-plane)"""
    lib().orc_set_combined_weights(float(w_point), float(w_plane))


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def get_threads() -> int:
    return int(lib().orc_get_threads())


def _pts(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    assert a.ndim == 2 and a.shape[1] == 3
    return a


class KDTree:
    """fp64 kd-tree over fp32 points (median split on the widest axis, leaf 16)."""

    def __init__(self, pts, leaf: int = 16):
        self.pts = _pts(pts)          # kept alive: the C tree references it
        self.n = self.pts.shape[0]
        self.h = lib().orc_kd_build(self.pts, self.n, int(leaf))

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib is not None:
            _lib.orc_kd_free(h)
            self.h = None


def knn(target, queries_f64, k: int = 1, max_dist: float = math.inf, tree: KDTree | None = None,
        brute: bool = False):
    """k nearest targets of fp64 queries; returns (idx int64 [m,k], d2 float64 [m,k])."""
    tgt = tree.pts if tree is not None else _pts(target)
    q = np.ascontiguousarray(queries_f64, dtype=np.float64).reshape(-1, 3)
    m = q.shape[0]
    idx = np.empty((m, k), np.int64)
    d2 = np.empty((m, k), np.float64)
    h = None if brute else (tree.h if tree is not None else None)
    if not brute and tree is None:
        tree = KDTree(tgt)
        h = tree.h
    bound2 = max_dist * max_dist if math.isfinite(max_dist) else math.inf
    rc = lib().orc_knn(h, tgt, tgt.shape[0], q, m, int(k), bound2, idx, d2)
    assert rc == 0
    return idx, d2


def transform(pose, pts) -> np.ndarray:
    p = _pts(pts)
    out = np.empty((p.shape[0], 3), np.float64)
    lib().orc_transform(np.ascontiguousarray(pose, np.float64).reshape(16), p, p.shape[0], out)
    return out


@dataclass
class System:
    H: np.ndarray
    g: np.ndarray
    sse: float
    count: int
    Habs: np.ndarray
    gabs: np.ndarray
    corr_idx: np.ndarray | None = None
    corr_d2: np.ndarray | None = None
    corr_d2nd: np.ndarray | None = None


def icp_system(target, normals, source, pose, metric: str, max_dist: float, tree: KDTree | None = None,
               brute: bool = False, want_corr: bool = True) -> System:
    tgt = tree.pts if tree is not None else _pts(target)
    nrm = None if normals is None else _pts(normals)
    src = _pts(source)
    if tree is None and not brute:
        tree = KDTree(tgt)
    h = None if brute else tree.h
    H = np.zeros(36); g = np.zeros(6); Ha = np.zeros(36); ga = np.zeros(6)
    sse = C.c_double(); cnt = C.c_int64()
    m = src.shape[0]
    ci = np.empty(m, np.int64) if want_corr else None
    cd = np.empty(m, np.float64) if want_corr else None
    cd2 = np.empty(m, np.float64) if want_corr else None
    rc = lib().orc_icp_system(h, tgt, nrm, tgt.shape[0], src, m, np.ascontiguousarray(pose, np.float64).reshape(16),
                              METRICS[metric], float(max_dist), H, g, C.byref(sse), C.byref(cnt), Ha, ga, ci, cd, cd2)
    if rc:
        raise ValueError(f"orc_icp_system rc={rc}")
    return System(H.reshape(6, 6), g, sse.value, cnt.value, Ha.reshape(6, 6), ga, ci, cd, cd2)


def icp_system_from_corr(target, normals, source, pose, metric: str, corr) -> System:
    tgt = _pts(target)
    nrm = None if normals is None else _pts(normals)
    src = _pts(source)
    H = np.zeros(36); g = np.zeros(6); Ha = np.zeros(36); ga = np.zeros(6)
    sse = C.c_double(); cnt = C.c_int64()
    rc = lib().orc_icp_system_from_corr(tgt, nrm, tgt.shape[0], src, src.shape[0],
                                        np.ascontiguousarray(pose, np.float64).reshape(16), METRICS[metric],
                                        np.ascontiguousarray(corr, np.int32), H, g, C.byref(sse), C.byref(cnt), Ha, ga)
    if rc:
        raise ValueError(f"orc_icp_system_from_corr rc={rc}")
    return System(H.reshape(6, 6), g, sse.value, cnt.value, Ha.reshape(6, 6), ga)


def rodrigues(alpha) -> np.ndarray:
    R = np.empty(9)
    lib().orc_rodrigues(np.ascontiguousarray(alpha, np.float64), R)
    return R.reshape(3, 3)


def solve_update(H, g, count: int, pose_in):
    pose_out = np.empty(16); x = np.empty(6)
    th = C.c_double(); tn = C.c_double()
    st = lib().orc_solve_update(np.ascontiguousarray(H, np.float64).reshape(36), np.ascontiguousarray(g, np.float64),
                                int(count), np.ascontiguousarray(pose_in, np.float64).reshape(16), pose_out, x,
                                C.byref(th), C.byref(tn))
    return st, pose_out.reshape(4, 4), x, th.value, tn.value


@dataclass
class RunResult:
    pose: np.ndarray
    rmse: float
    n_corr: int
    iterations: int
    converged: bool
    status: int
    iter_log: np.ndarray
    H_log: np.ndarray
    g_log: np.ndarray
    pose_log: np.ndarray


def icp_run(target, normals, source, metric: str, max_iters: int, max_dist: float, pose_init=None,
            rot_tol: float = 0.0, trans_tol: float = 0.0, tree: KDTree | None = None, brute: bool = False) -> RunResult:
    tgt = tree.pts if tree is not None else _pts(target)
    nrm = None if normals is None else _pts(normals)
    src = _pts(source)
    if tree is None and not brute:
        tree = KDTree(tgt)
    h = None if brute else tree.h
    P0 = np.eye(4) if pose_init is None else np.asarray(pose_init, np.float64)
    pose = np.empty(16); rmse = C.c_double(); nc = C.c_int64()
    it = C.c_int32(); cv = C.c_int32(); st = C.c_int32()
    K = max(int(max_iters), 1)
    log = np.zeros(2 * K); Hl = np.zeros(36 * K); gl = np.zeros(6 * K); Pl = np.zeros(16 * K)
    rc = lib().orc_icp_run(h, tgt, nrm, tgt.shape[0], src, src.shape[0], np.ascontiguousarray(P0).reshape(16),
                           METRICS[metric], int(max_iters), float(max_dist), float(rot_tol), float(trans_tol),
                           pose, C.byref(rmse), C.byref(nc), C.byref(it), C.byref(cv), C.byref(st), log, Hl, gl, Pl)
    if rc:
        raise ValueError(f"orc_icp_run rc={rc}")
    n_it = it.value
    return RunResult(pose.reshape(4, 4), rmse.value, nc.value, n_it, bool(cv.value), st.value,
                     log.reshape(K, 2)[:n_it], Hl.reshape(K, 6, 6)[:n_it], gl.reshape(K, 6)[:n_it],
                     Pl.reshape(K, 4, 4)[:n_it])


@dataclass
class ProjSystem(System):
    uv: np.ndarray | None = None


def _intr(intr) -> np.ndarray:
    """intr = (width, height, fx, fy, cx, cy) -> (w, h, [fx, fy, cx, cy])"""
    w, h, fx, fy, cx, cy = intr
    return int(w), int(h), np.array([fx, fy, cx, cy], np.float64)


def proj_system(target, normals, intr, source, pose, metric: str, max_dist: float) -> ProjSystem:
    """projective correspondences (R23-R26) + the normal equations of one iteration;
    target: organised [w*h, 3] in row-major pixel order"""
    tgt = _pts(target)
    nrm = None if normals is None else _pts(normals)
    src = _pts(source)
    w, h, K = _intr(intr)
    assert tgt.shape[0] == w * h
    m = src.shape[0]
    H = np.zeros(36); g = np.zeros(6); Ha = np.zeros(36); ga = np.zeros(6)
    sse = C.c_double(); cnt = C.c_int64()
    ci = np.empty(m, np.int64); cd = np.empty(m, np.float64); uv = np.empty(2 * m, np.float64)
    rc = lib().orc_proj_system(tgt, nrm, w, h, K, src, m, np.ascontiguousarray(pose, np.float64).reshape(16),
                               METRICS[metric], float(max_dist), H, g, C.byref(sse), C.byref(cnt), Ha, ga, ci, cd, uv)
    if rc:
        raise ValueError(f"orc_proj_system rc={rc}")
    return ProjSystem(H.reshape(6, 6), g, sse.value, cnt.value, Ha.reshape(6, 6), ga, ci, cd, None, uv.reshape(m, 2))


def proj_run(target, normals, intr, source, metric: str, max_iters: int, max_dist: float, pose_init=None,
             rot_tol: float = 0.0, trans_tol: float = 0.0) -> RunResult:
    tgt = _pts(target)
    nrm = None if normals is None else _pts(normals)
    src = _pts(source)
    w, h, K = _intr(intr)
    assert tgt.shape[0] == w * h
    P0 = np.eye(4) if pose_init is None else np.asarray(pose_init, np.float64)
    pose = np.empty(16); rmse = C.c_double(); nc = C.c_int64()
    it = C.c_int32(); cv = C.c_int32(); st = C.c_int32()
    n = max(int(max_iters), 1)
    log = np.zeros(2 * n); Hl = np.zeros(36 * n); gl = np.zeros(6 * n); Pl = np.zeros(16 * n)
    rc = lib().orc_proj_run(tgt, nrm, w, h, K, src, src.shape[0], np.ascontiguousarray(P0).reshape(16),
                            METRICS[metric], int(max_iters), float(max_dist), float(rot_tol), float(trans_tol),
                            pose, C.byref(rmse), C.byref(nc), C.byref(it), C.byref(cv), C.byref(st), log, Hl, gl, Pl)
    if rc:
        raise ValueError(f"orc_proj_run rc={rc}")
    n_it = it.value
    return RunResult(pose.reshape(4, 4), rmse.value, nc.value, n_it, bool(cv.value), st.value,
                     log.reshape(n, 2)[:n_it], Hl.reshape(n, 6, 6)[:n_it], gl.reshape(n, 6)[:n_it],
                     Pl.reshape(n, 4, 4)[:n_it])


def pca_normals(pts, k: int = 10, view=(0.0, 0.0, 0.0), tree: KDTree | None = None, brute: bool = False):
    p = tree.pts if tree is not None else _pts(pts)
    if tree is None and not brute:
        tree = KDTree(p)
    h = None if brute else tree.h
    out = np.empty_like(p)
    curv = np.empty(p.shape[0], np.float32)
    rc = lib().orc_pca_normals(h, p, p.shape[0], int(k), np.asarray(view, np.float64), out, curv)
    assert rc == 0
    return out, curv


def voxel_downsample(pts, bin_size: float, origin=(0.0, 0.0, 0.0), normals=None):
    """voxel-grid downsampling (R27-R29): returns (points [b,3] f32, normals [b,3] or
    None, keys [b,3] int64) in ascending key order; raises on a key outside int32"""
    p = _pts(pts)
    nrm = None if normals is None else _pts(normals)
    n = p.shape[0]
    op = np.empty((max(n, 1), 3), np.float32)
    on = np.empty((max(n, 1), 3), np.float32) if nrm is not None else None
    ok = np.empty((max(n, 1), 3), np.int64)
    nb = lib().orc_voxel_downsample(p, nrm, n, float(bin_size), np.asarray(origin, np.float64), op, on, ok)
    if nb < 0:
        raise ValueError("voxel key outside int32 or not finite")
    return op[:nb], (on[:nb] if on is not None else None), ok[:nb]
