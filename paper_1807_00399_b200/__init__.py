"""paper_1807_00399_b200 -- thin Python binding over libcil.so (include/cil.h).

The binding only marshals arguments: torch tensors provide device memory and the CUDA
stream (torch.cuda.current_stream() by default); every step of the ICP hot path runs in
the library's own sm_100a kernels.  There is no CPU fallback: importing this package
fails loudly if libcil.so is missing, and every call raises CilError on failure.

Function names match the C ABI (cil_target_build, cil_nn_query, cil_icp_workspace_bytes,
cil_icp_iterate, cil_icp_run, cil_target_free).
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcil.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libcil.so not built at {LIB_PATH}: run `make` or __graft_entry__.build(); "
                      "there is no CPU fallback for the ICP hot path")

_lib = C.CDLL(LIB_PATH)

# ---------------------------------------------------------------- status / structs
CIL_OK = 0
CIL_ERR_INVALID_ARG = 1
CIL_ERR_EMPTY_TARGET = 2
CIL_ERR_NO_NORMALS = 3
CIL_ERR_CUDA = 4
CIL_ERR_OOM = 5
CIL_ERR_WORKSPACE = 6
CIL_ERR_DEGENERATE = 16
CIL_NO_CORRESPONDENCES = 17
CIL_INDEX_BVH = 0
CIL_INDEX_GRID = 1
CIL_POINT_TO_POINT = 0
CIL_POINT_TO_PLANE = 1
CIL_COMBINED = 2
METRICS = {"point_to_point": CIL_POINT_TO_POINT, "point_to_plane": CIL_POINT_TO_PLANE, "combined": CIL_COMBINED}

EXPORTED = ["cil_target_build", "cil_target_free", "cil_target_get_info", "cil_nn_query", "cil_estimate_normals",
            "cil_icp_workspace_bytes", "cil_icp_iterate", "cil_icp_run", "cil_status_string",
            "cil_last_error", "cil_version", "cil_launch_count", "cil_profile_enable", "cil_profile_read",
            "cil_debug_set_flags", "cil_debug_engine_trace", "cil_debug_set_cert_skin",
            "cil_proj_workspace_bytes", "cil_proj_iterate", "cil_proj_run", "cil_debug_timestamps",
            "cil_voxel_downsample", "cil_icp_shard_begin", "cil_icp_shard_accumulate", "cil_icp_shard_finish",
            "cil_icp_shard_result", "cil_icp_align_host"]


class cil_index_params(C.Structure):
    _fields_ = [("leaf_size", C.c_int32), ("index_kind", C.c_int32), ("grid_points", C.c_float),
                ("reserved", C.c_int32 * 5)]


class cil_icp_params(C.Structure):
    _fields_ = [("metric", C.c_int32), ("max_iters", C.c_int32), ("max_corr_dist", C.c_double),
                ("rot_tol", C.c_double), ("trans_tol", C.c_double), ("w_point", C.c_double),
                ("w_plane", C.c_double)]


class cil_icp_result(C.Structure):
    _fields_ = [("pose", C.c_double * 16), ("rmse", C.c_double), ("n_corr", C.c_int64),
                ("iterations", C.c_int32), ("converged", C.c_int32), ("status", C.c_int32), ("pad", C.c_int32)]


class cil_icp_system(C.Structure):
    _fields_ = [("H", C.c_double * 36), ("g", C.c_double * 6), ("x", C.c_double * 6), ("sse", C.c_double),
                ("n_corr", C.c_int64), ("status", C.c_int32), ("pad", C.c_int32)]


class cil_profile_stats(C.Structure):
    _fields_ = [("build_ms", C.c_double), ("nn_ms", C.c_double), ("acc_ms", C.c_double), ("query_ms", C.c_double),
                ("n_build", C.c_int64), ("n_nn", C.c_int64), ("n_acc", C.c_int64), ("n_query", C.c_int64),
                ("sel_ms", C.c_double), ("n_sel", C.c_int64)]


class cil_intrinsics(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double)]


def make_intrinsics(width: int, height: int, fx: float, fy: float, cx: float, cy: float) -> cil_intrinsics:
    k = cil_intrinsics()
    k.width, k.height = int(width), int(height)
    k.fx, k.fy, k.cx, k.cy = float(fx), float(fy), float(cx), float(cy)
    return k


class cil_target_info(C.Structure):
    _fields_ = [("n", C.c_int64), ("n_leaves", C.c_int64), ("n_nodes", C.c_int64), ("leaf_size", C.c_int32),
                ("has_normals", C.c_int32), ("device_bytes", C.c_int64), ("index_kind", C.c_int32),
                ("pad", C.c_int32)]


_vp, _i64, _sz = C.c_void_p, C.c_int64, C.c_size_t
_lib.cil_target_build.restype = C.c_int
_lib.cil_target_build.argtypes = [_vp, _vp, _i64, C.POINTER(cil_index_params), _vp, C.POINTER(_vp)]
_lib.cil_target_free.restype = C.c_int
_lib.cil_target_free.argtypes = [_vp, _vp]
_lib.cil_target_get_info.restype = C.c_int
_lib.cil_target_get_info.argtypes = [_vp, C.POINTER(cil_target_info)]
_lib.cil_nn_query.restype = C.c_int
_lib.cil_nn_query.argtypes = [_vp, _vp, _i64, C.c_float, _vp, _vp, _vp]
_lib.cil_estimate_normals.restype = C.c_int
_lib.cil_estimate_normals.argtypes = [_vp, C.c_int32, C.POINTER(C.c_double * 3), _vp, _vp, _vp]
_lib.cil_icp_workspace_bytes.restype = _sz
_lib.cil_icp_workspace_bytes.argtypes = [_i64, C.POINTER(cil_icp_params)]
_lib.cil_icp_iterate.restype = C.c_int
_lib.cil_icp_iterate.argtypes = [_vp, _vp, _i64, _vp, C.POINTER(cil_icp_params), _vp, _sz, _vp, _vp, _vp, _vp, _vp]
_lib.cil_icp_run.restype = C.c_int
_lib.cil_icp_run.argtypes = [_vp, _vp, _i64, _vp, C.POINTER(cil_icp_params), _vp, _sz, _vp, _vp, _vp]
_lib.cil_icp_align_host.restype = C.c_int
_lib.cil_icp_align_host.argtypes = [_vp, _vp, _i64, _vp, _i64, _vp, C.POINTER(cil_icp_params), C.POINTER(cil_index_params),
                                    C.POINTER(cil_icp_result), _vp]
_lib.cil_proj_workspace_bytes.restype = _sz
_lib.cil_proj_workspace_bytes.argtypes = [_i64, C.POINTER(cil_icp_params)]
_lib.cil_proj_iterate.restype = C.c_int
_lib.cil_proj_iterate.argtypes = [_vp, _vp, C.POINTER(cil_intrinsics), _vp, _i64, _vp, C.POINTER(cil_icp_params), _vp,
                                  _sz, _vp, _vp, _vp, _vp, _vp]
_lib.cil_proj_run.restype = C.c_int
_lib.cil_proj_run.argtypes = [_vp, _vp, C.POINTER(cil_intrinsics), _vp, _i64, _vp, C.POINTER(cil_icp_params), _vp, _sz,
                              _vp, _vp, _vp]
_lib.cil_icp_shard_begin.restype = C.c_int
_lib.cil_icp_shard_begin.argtypes = [_vp, _vp, _i64, _vp, C.POINTER(cil_icp_params), _vp, _sz, _vp, _vp]
_lib.cil_icp_shard_accumulate.restype = C.c_int
_lib.cil_icp_shard_accumulate.argtypes = [_vp, _vp, _i64, C.POINTER(cil_icp_params), _vp, _sz, _vp, _vp]
_lib.cil_icp_shard_finish.restype = C.c_int
_lib.cil_icp_shard_finish.argtypes = [_vp, _i64, C.POINTER(cil_icp_params), _vp, _sz, _vp, _vp, _vp]
_lib.cil_icp_shard_result.restype = C.c_int
_lib.cil_icp_shard_result.argtypes = [_vp, _vp, _vp]
_lib.cil_voxel_downsample.restype = C.c_int
_lib.cil_voxel_downsample.argtypes = [_vp, _vp, _i64, C.c_double, C.POINTER(C.c_double * 3), _vp, _vp, _vp, _vp]
_lib.cil_status_string.restype = C.c_char_p
_lib.cil_status_string.argtypes = [C.c_int]
_lib.cil_last_error.restype = C.c_char_p
_lib.cil_version.restype = C.c_char_p
_lib.cil_launch_count.restype = C.c_uint64


_lib.cil_profile_enable.restype = C.c_int
_lib.cil_profile_enable.argtypes = [C.c_int]
_lib.cil_profile_read.restype = C.c_int
_lib.cil_profile_read.argtypes = [C.POINTER(cil_profile_stats)]
_lib.cil_debug_set_flags.restype = C.c_int
_lib.cil_debug_set_flags.argtypes = [C.c_uint32]
_lib.cil_debug_engine_trace.restype = C.c_int
_lib.cil_debug_engine_trace.argtypes = [C.c_void_p]
_lib.cil_debug_timestamps.restype = C.c_int
_lib.cil_debug_timestamps.argtypes = [C.c_void_p]
_lib.cil_debug_set_cert_skin.restype = C.c_int
_lib.cil_debug_set_cert_skin.argtypes = [C.c_double, C.c_double, C.c_double]

# Byte offsets into the ICP workspace (csrc/icp.cu ws_layout, IcpState) -- diagnostics only.
WS_STATE_SEARCHED = 176       # int64: sum over executed iterations of the search-list size
WS_STATE_PCERT = 184          # int64: sum over executed iterations of point-certified points


def set_certificates(on: bool = True) -> None:
    """cil_icp_run: certified warm start on (default) or a full search every iteration (diagnostics)."""
    _check(_lib.cil_debug_set_flags(0 if on else 1), "cil_debug_set_flags")


def set_debug_flags(flags: int) -> None:
    """cil_debug_set_flags (diagnostics): bit 0 no certified warm start, bits 1-2 engine mode,
    bit 3 no point certificate, bit 4 caller's source order, bit 5 Morton source order,
    bit 6 no small-problem (brute-force) path"""
    _check(_lib.cil_debug_set_flags(int(flags)), "cil_debug_set_flags")


def set_cert_skin(min_frac: float = 0.001, max_frac: float = 0.005, kappa: float = 16.0) -> None:
    """certificate skin of cil_icp_run: g = clamp(kappa * last-step displacement, min, max) x max_corr_dist"""
    _check(_lib.cil_debug_set_cert_skin(float(min_frac), float(max_frac), float(kappa)), "cil_debug_set_cert_skin")


def run_point_certified(ws: torch.Tensor) -> int:
    """points kept by the point certificate in cil_icp_run (sum over iterations; diagnostics)"""
    return int(ws[WS_STATE_PCERT:WS_STATE_PCERT + 8].cpu().view(torch.int64).item())


def run_searched(ws: torch.Tensor) -> int:
    """number of full searches cil_icp_run did (sum over iterations), read from the workspace"""
    return int(ws[WS_STATE_SEARCHED:WS_STATE_SEARCHED + 8].cpu().view(torch.int64).item())


def debug_timestamps(buf: torch.Tensor | None) -> None:
    """per-iteration %globaltimer stamps of the ICP kernels into buf (int64 [iters, 8], filled
    with -1 by the caller); None switches them off (diagnostics)"""
    _check(_lib.cil_debug_timestamps(None if buf is None else buf.data_ptr()), "cil_debug_timestamps")


def profile_enable(on: bool = True) -> None:
    """per-launch CUDA-event timing inside the library (diagnostics)"""
    _check(_lib.cil_profile_enable(1 if on else 0), "cil_profile_enable")


def profile_read() -> dict:
    st = cil_profile_stats()
    _check(_lib.cil_profile_read(C.byref(st)), "cil_profile_read")
    return {k: getattr(st, k) for k, _ in cil_profile_stats._fields_}


def launch_count() -> int:
    """kernels enqueued by libcil.so in this process so far"""
    return int(_lib.cil_launch_count())


class CilError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = f"{where}: {_lib.cil_status_string(status).decode()} ({_lib.cil_last_error().decode()})"
        super().__init__(msg)


def _check(rc: int, where: str) -> None:
    if rc != CIL_OK:
        raise CilError(rc, where)


def version() -> str:
    return _lib.cil_version().decode()


def lib() -> C.CDLL:
    return _lib


def _stream_ptr(stream) -> int | None:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _pts(t: torch.Tensor, name: str) -> torch.Tensor:
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32 and t.dim() == 2
            and t.shape[1] == 3 and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous CUDA float32 tensor of shape [n, 3]")
    return t


def make_params(metric: str | int = "point_to_plane", max_iters: int = 1, max_corr_dist: float = math.inf,
                rot_tol: float = 0.0, trans_tol: float = 0.0, w_point: float = 0.0,
                w_plane: float = 0.0) -> cil_icp_params:
    p = cil_icp_params()
    p.metric = METRICS[metric] if isinstance(metric, str) else int(metric)
    p.max_iters = int(max_iters)
    p.max_corr_dist = float(max_corr_dist)
    p.rot_tol = float(rot_tol)
    p.trans_tol = float(trans_tol)
    p.w_point = float(w_point)
    p.w_plane = float(w_plane)
    return p


# ---------------------------------------------------------------- ABI-named entry points
class Target:
    """Owning handle of a cil_target (built on the GPU, immutable)."""

    def __init__(self, handle: int, n: int, keep=(), stream=None):
        self.handle = handle
        self.n = n
        self._keep = keep
        self._streams = {}
        self.use(stream)                      # the build stream

    def info(self) -> cil_target_info:
        inf = cil_target_info()
        _check(_lib.cil_target_get_info(self.handle, C.byref(inf)), "cil_target_get_info")
        return inf

    def use(self, stream=None) -> int:
        """the stream pointer of a call on this target; remembers the stream, so that free()
        orders the release after the work of every stream the target was used on"""
        st = torch.cuda.current_stream() if stream is None else stream
        self._streams[st.cuda_stream] = st
        return st.cuda_stream

    def _release(self, stream) -> int:
        st = torch.cuda.current_stream() if stream is None else stream
        for ptr, other in self._streams.items():
            if ptr != st.cuda_stream:
                ev = torch.cuda.Event()
                ev.record(other)
                st.wait_event(ev)
        self._streams = {}
        return st.cuda_stream

    def free(self, stream=None) -> None:
        """stream-ordered release on `stream` (default: the current stream), after the work
        already enqueued on every stream this target was used on.  Free targets explicitly;
        garbage collection does the same from whatever stream is current then."""
        if self.handle:
            _check(_lib.cil_target_free(self.handle, self._release(stream)), "cil_target_free")
            self.handle = None

    def __del__(self):
        try:
            if self.handle and torch.cuda.is_available():
                _lib.cil_target_free(self.handle, self._release(None))
        except Exception:
            pass


def cil_target_build(pts: torch.Tensor, normals: torch.Tensor | None = None, leaf_size: int = 0,
                     stream=None, index: str = "bvh", grid_points: float = 0.0) -> Target:
    _pts(pts, "pts")
    if normals is not None:
        _pts(normals, "normals")
        if normals.shape != pts.shape:
            raise ValueError("normals must match pts")
    prm = cil_index_params()
    prm.leaf_size = int(leaf_size)
    prm.index_kind = {"bvh": CIL_INDEX_BVH, "grid": CIL_INDEX_GRID}[index]
    prm.grid_points = float(grid_points)
    h = _vp()
    _check(_lib.cil_target_build(_ptr(pts), _ptr(normals), pts.shape[0], C.byref(prm), _stream_ptr(stream),
                                 C.byref(h)), "cil_target_build")
    return Target(h.value, pts.shape[0], stream=stream)


def cil_target_free(t: Target, stream=None) -> None:
    t.free(stream)


def cil_nn_query(t: Target, queries: torch.Tensor, max_dist: float = math.inf, stream=None,
                 idx: torch.Tensor | None = None, sqdist: torch.Tensor | None = None):
    _pts(queries, "queries")
    m = queries.shape[0]
    dev = queries.device
    if idx is None:
        idx = torch.empty(m, dtype=torch.int32, device=dev)
    if sqdist is None:
        sqdist = torch.empty(m, dtype=torch.float32, device=dev)
    _check(_lib.cil_nn_query(t.handle, _ptr(queries), m, float(max_dist), _ptr(idx), _ptr(sqdist),
                             t.use(stream)), "cil_nn_query")
    return idx, sqdist


def cil_estimate_normals(t: Target, k: int = 10, view=(0.0, 0.0, 0.0), stream=None, want_curvature: bool = False,
                         device="cuda"):
    """PCA normals of the target over its k nearest neighbours, oriented towards `view`.
    Returns (normals [n,3] fp32 device tensor in original order, curvature [n] or None)."""
    nrm = torch.empty((t.n, 3), dtype=torch.float32, device=device)
    cur = torch.empty(t.n, dtype=torch.float32, device=device) if want_curvature else None
    v = (C.c_double * 3)(*[float(x) for x in view])
    _check(_lib.cil_estimate_normals(t.handle, int(k), C.byref(v), _ptr(nrm), _ptr(cur), t.use(stream)),
           "cil_estimate_normals")
    return nrm, cur


def cil_icp_workspace_bytes(m: int, params: cil_icp_params) -> int:
    return int(_lib.cil_icp_workspace_bytes(int(m), C.byref(params)))


def alloc_workspace(m: int, params: cil_icp_params, device="cuda") -> torch.Tensor:
    nb = cil_icp_workspace_bytes(m, params)
    if nb == 0:
        raise ValueError("invalid workspace request")
    return torch.empty(nb, dtype=torch.uint8, device=device)   # caching allocator: >= 512-B aligned


def _struct_tensor(ctype, device) -> torch.Tensor:
    return torch.zeros(C.sizeof(ctype), dtype=torch.uint8, device=device)


def read_struct(t: torch.Tensor, ctype):
    return ctype.from_buffer_copy(t.cpu().numpy().tobytes())


def cil_icp_iterate(t: Target, src: torch.Tensor, pose_in: torch.Tensor, params: cil_icp_params,
                    ws: torch.Tensor | None = None, pose_out: torch.Tensor | None = None,
                    want_sys: bool = True, want_corr: bool = False, stream=None):
    """One stateless ICP iteration.  Returns (pose_out [4,4] f64 device, sys_bytes device
    tensor or None, corr_idx or None, corr_sqdist or None)."""
    _pts(src, "src")
    m = src.shape[0]
    dev = src.device
    if ws is None:
        ws = alloc_workspace(m, params, dev)
    if pose_out is None:
        pose_out = torch.empty((4, 4), dtype=torch.float64, device=dev)
    sys_t = _struct_tensor(cil_icp_system, dev) if want_sys else None
    ci = torch.empty(m, dtype=torch.int32, device=dev) if want_corr else None
    cd = torch.empty(m, dtype=torch.float32, device=dev) if want_corr else None
    _check(_lib.cil_icp_iterate(t.handle, _ptr(src), m, _ptr(pose_in), C.byref(params), _ptr(ws), ws.numel(),
                                _ptr(pose_out), _ptr(sys_t), _ptr(ci), _ptr(cd), t.use(stream)),
           "cil_icp_iterate")
    return pose_out, sys_t, ci, cd


def cil_icp_run(t: Target, src: torch.Tensor, pose_init: torch.Tensor, params: cil_icp_params,
                ws: torch.Tensor | None = None, res: torch.Tensor | None = None, iter_log: torch.Tensor | None = None,
                want_log: bool = True, stream=None):
    """The device-resident ICP loop.  Returns (res_bytes device tensor, iter_log [max_iters,2] or None)."""
    _pts(src, "src")
    m = src.shape[0]
    dev = src.device
    if ws is None:
        ws = alloc_workspace(m, params, dev)
    if res is None:
        res = _struct_tensor(cil_icp_result, dev)
    if iter_log is None and want_log:
        iter_log = torch.empty((params.max_iters, 2), dtype=torch.float64, device=dev)
    _check(_lib.cil_icp_run(t.handle, _ptr(src), m, _ptr(pose_init), C.byref(params), _ptr(ws), ws.numel(),
                            _ptr(res), _ptr(iter_log), t.use(stream)), "cil_icp_run")
    return res, iter_log


def _host_pts(t, name: str) -> torch.Tensor:
    t = torch.as_tensor(t)
    if t.is_cuda or t.dtype != torch.float32 or t.dim() != 2 or t.shape[1] != 3 or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous HOST float32 array of shape [n, 3]")
    return t


def cil_icp_align_host(target, normals, source, pose_init=None, params: cil_icp_params | None = None,
                       leaf_size: int = 0, index: str = "bvh", stream=None) -> "Result":
    """One frame pair end to end from HOST buffers through the C ABI (cil_icp_align_host): the
    copies in, the index build, the device-resident loop and the result copy all happen inside
    the library call.  Inputs: CPU float32 [n, 3] tensors / arrays (pinned tensors make the
    copies asynchronous), pose_init a CPU float64 [4, 4] or None (identity).  Synchronous."""
    ht = _host_pts(target, "target")
    hn = _host_pts(normals, "normals") if normals is not None else None
    hs = _host_pts(source, "source")
    if hn is not None and hn.shape != ht.shape:
        raise ValueError("normals must match target")
    hp = None
    if pose_init is not None:
        hp = torch.as_tensor(pose_init, dtype=torch.float64).contiguous()
        if hp.is_cuda or hp.shape != (4, 4):
            raise ValueError("pose_init must be a HOST float64 [4, 4]")
    ip = cil_index_params()
    ip.leaf_size = int(leaf_size)
    ip.index_kind = {"bvh": CIL_INDEX_BVH, "grid": CIL_INDEX_GRID}[index]
    r = cil_icp_result()
    _check(_lib.cil_icp_align_host(_ptr(ht), _ptr(hn), ht.shape[0], _ptr(hs), hs.shape[0], _ptr(hp),
                                   C.byref(params if params is not None else make_params()), C.byref(ip), C.byref(r),
                                   _stream_ptr(stream)), "cil_icp_align_host")
    return Result(np.array(r.pose).reshape(4, 4), r.rmse, r.n_corr, r.iterations, bool(r.converged), r.status)


# ---------------------------------------------------------------- projective engine (NEXT-2)
def _organised(tgt: torch.Tensor, K: cil_intrinsics, name: str) -> None:
    _pts(tgt, name)
    if tgt.shape[0] != K.width * K.height:
        raise ValueError(f"{name} must hold width*height = {K.width * K.height} points, got {tgt.shape[0]}")


def cil_proj_workspace_bytes(m: int, params: cil_icp_params) -> int:
    return int(_lib.cil_proj_workspace_bytes(int(m), C.byref(params)))


def cil_proj_iterate(tgt: torch.Tensor, tgt_normals: torch.Tensor | None, K: cil_intrinsics, src: torch.Tensor,
                     pose_in: torch.Tensor, params: cil_icp_params, ws: torch.Tensor | None = None,
                     pose_out: torch.Tensor | None = None, want_sys: bool = True, want_corr: bool = False,
                     stream=None):
    """One projective-association ICP iteration on an organised target (tgt [w*h, 3] row-major
    pixels).  Returns (pose_out, sys_bytes or None, corr_idx or None, corr_sqdist or None)."""
    _organised(tgt, K, "tgt")
    if tgt_normals is not None:
        _organised(tgt_normals, K, "tgt_normals")
    _pts(src, "src")
    m = src.shape[0]
    dev = src.device
    if ws is None:
        ws = torch.empty(cil_proj_workspace_bytes(m, params), dtype=torch.uint8, device=dev)
    if pose_out is None:
        pose_out = torch.empty((4, 4), dtype=torch.float64, device=dev)
    sys_t = _struct_tensor(cil_icp_system, dev) if want_sys else None
    ci = torch.empty(m, dtype=torch.int32, device=dev) if want_corr else None
    cd = torch.empty(m, dtype=torch.float32, device=dev) if want_corr else None
    _check(_lib.cil_proj_iterate(_ptr(tgt), _ptr(tgt_normals), C.byref(K), _ptr(src), m, _ptr(pose_in),
                                 C.byref(params), _ptr(ws), ws.numel(), _ptr(pose_out), _ptr(sys_t), _ptr(ci),
                                 _ptr(cd), _stream_ptr(stream)), "cil_proj_iterate")
    return pose_out, sys_t, ci, cd


def cil_proj_run(tgt: torch.Tensor, tgt_normals: torch.Tensor | None, K: cil_intrinsics, src: torch.Tensor,
                 pose_init: torch.Tensor, params: cil_icp_params, ws: torch.Tensor | None = None,
                 res: torch.Tensor | None = None, iter_log: torch.Tensor | None = None, want_log: bool = True,
                 stream=None):
    """The device-resident projective ICP loop.  Returns (res_bytes, iter_log or None)."""
    _organised(tgt, K, "tgt")
    if tgt_normals is not None:
        _organised(tgt_normals, K, "tgt_normals")
    _pts(src, "src")
    m = src.shape[0]
    dev = src.device
    if ws is None:
        ws = torch.empty(cil_proj_workspace_bytes(m, params), dtype=torch.uint8, device=dev)
    if res is None:
        res = _struct_tensor(cil_icp_result, dev)
    if iter_log is None and want_log:
        iter_log = torch.empty((params.max_iters, 2), dtype=torch.float64, device=dev)
    _check(_lib.cil_proj_run(_ptr(tgt), _ptr(tgt_normals), C.byref(K), _ptr(src), m, _ptr(pose_init),
                             C.byref(params), _ptr(ws), ws.numel(), _ptr(res), _ptr(iter_log), _stream_ptr(stream)),
           "cil_proj_run")
    return res, iter_log


# ---------------------------------------------------------------- one problem across ranks
class ShardRun:
    """One rank's part of an ICP problem whose source is split across ranks (C ABI
    cil_icp_shard_*).  accumulate() -> the caller all-reduces .sums -> finish()."""

    def __init__(self, t: Target, src_shard: torch.Tensor, pose_init: torch.Tensor, params: cil_icp_params,
                 want_log: bool = True, stream=None, ws: torch.Tensor | None = None):
        _pts(src_shard, "src_shard")
        self.t, self.src, self.params, self.stream = t, src_shard, params, stream
        self.m = src_shard.shape[0]
        dev = src_shard.device
        self.ws = ws if ws is not None else alloc_workspace(self.m, params, dev)
        self.sums = torch.zeros(32, dtype=torch.float64, device=dev)
        self.iter_log = torch.empty((params.max_iters, 2), dtype=torch.float64, device=dev) if want_log else None
        _check(_lib.cil_icp_shard_begin(t.handle, _ptr(src_shard), self.m, _ptr(pose_init), C.byref(params),
                                        _ptr(self.ws), self.ws.numel(), _ptr(self.iter_log), t.use(stream)),
               "cil_icp_shard_begin")

    def accumulate(self) -> torch.Tensor:
        _check(_lib.cil_icp_shard_accumulate(self.t.handle, _ptr(self.src), self.m, C.byref(self.params),
                                             _ptr(self.ws), self.ws.numel(), _ptr(self.sums),
                                             self.t.use(self.stream)), "cil_icp_shard_accumulate")
        return self.sums

    def finish(self, reduced: torch.Tensor | None = None) -> None:
        r = self.sums if reduced is None else reduced
        _check(_lib.cil_icp_shard_finish(self.t.handle, self.m, C.byref(self.params), _ptr(self.ws), self.ws.numel(),
                                         _ptr(r), _ptr(self.iter_log), _stream_ptr(self.stream)),
               "cil_icp_shard_finish")

    def result(self) -> torch.Tensor:
        res = _struct_tensor(cil_icp_result, self.ws.device)
        _check(_lib.cil_icp_shard_result(_ptr(self.ws), _ptr(res), _stream_ptr(self.stream)), "cil_icp_shard_result")
        return res


def icp_run_distributed(t: Target, src_shard: torch.Tensor, pose_init: torch.Tensor, params: cil_icp_params,
                        group=None, stream=None):
    """cil_icp_run over a source split across the ranks of torch.distributed `group`: one
    all-reduce of 32 fp64 sums per iteration (NCCL on GPUs).  Every rank gets the same pose."""
    import contextlib
    import torch.distributed as dist
    # every step runs on ONE stream, made current for the duration: the library calls use the
    # current stream and NCCL orders the all-reduce against the current stream (a non-current
    # `stream` would let the reduce read the sums before the accumulation wrote them)
    ctx = torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
    with ctx:
        run = ShardRun(t, src_shard, pose_init, params)
        for _ in range(params.max_iters):
            s = run.accumulate()
            dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
            run.finish()
        return run.result(), run.iter_log


# ---------------------------------------------------------------- voxel-grid downsampling (NEXT-4)
def cil_voxel_downsample(pts: torch.Tensor, bin_size: float, origin=(0.0, 0.0, 0.0),
                         normals: torch.Tensor | None = None, stream=None, sync: bool = True):
    """Voxel-grid downsampling on the GPU.  sync=True: returns (points [b,3], normals [b,3] or
    None) after reading the bin count; sync=False: returns the full-size buffers and the device
    int64 count tensor without synchronising."""
    _pts(pts, "pts")
    n = pts.shape[0]
    dev = pts.device
    if normals is not None:
        _pts(normals, "normals")
    out = torch.empty((max(n, 1), 3), dtype=torch.float32, device=dev)
    out_n = torch.empty((max(n, 1), 3), dtype=torch.float32, device=dev) if normals is not None else None
    cnt = torch.empty(1, dtype=torch.int64, device=dev)
    o = (C.c_double * 3)(*[float(v) for v in origin])
    _check(_lib.cil_voxel_downsample(_ptr(pts), _ptr(normals), n, float(bin_size), C.byref(o), _ptr(out), _ptr(out_n),
                                     _ptr(cnt), _stream_ptr(stream)), "cil_voxel_downsample")
    if not sync:
        return out, out_n, cnt
    nb = int(cnt.item())
    if nb < 0:
        raise CilError(CIL_ERR_INVALID_ARG, "cil_voxel_downsample: key not finite or axis span >= 2^21 bins")
    return out[:nb], (out_n[:nb] if out_n is not None else None)


# ---------------------------------------------------------------- decoded views
@dataclass
class System:
    H: np.ndarray
    g: np.ndarray
    x: np.ndarray
    sse: float
    n_corr: int
    status: int


@dataclass
class Result:
    pose: np.ndarray
    rmse: float
    n_corr: int
    iterations: int
    converged: bool
    status: int


def decode_system(t: torch.Tensor) -> System:
    s = read_struct(t, cil_icp_system)
    return System(np.array(s.H).reshape(6, 6), np.array(s.g), np.array(s.x), s.sse, s.n_corr, s.status)


def decode_result(t: torch.Tensor) -> Result:
    r = read_struct(t, cil_icp_result)
    return Result(np.array(r.pose).reshape(4, 4), r.rmse, r.n_corr, r.iterations, bool(r.converged), r.status)


def icp_align(target_pts, target_normals, source_pts, metric="point_to_plane", max_iters=30, max_corr_dist=0.05,
              pose_init=None, rot_tol=0.0, trans_tol=0.0, leaf_size=0, device="cuda", stream=None) -> Result:
    """End-to-end public call from HOST arrays (numpy or CPU tensors): host->device copies,
    target build, the device-resident ICP loop, and a device->host read of the result."""
    def to_dev(a):
        if a is None:
            return None
        ta = torch.as_tensor(a)
        return ta.to(device=device, dtype=torch.float32, non_blocking=True).contiguous()
    main = torch.cuda.current_stream(device) if stream is None else stream
    with torch.cuda.stream(main):
        tp, tn = to_dev(target_pts), to_dev(target_normals)
        side = torch.cuda.Stream(device=device)      # the source copy overlaps the index build
        side.wait_stream(main)
        with torch.cuda.stream(side):
            sp = to_dev(source_pts)
            P0 = torch.as_tensor(np.eye(4) if pose_init is None else np.asarray(pose_init, np.float64)).to(device)
        prm = make_params(metric, max_iters, max_corr_dist, rot_tol, trans_tol)
        tgt = cil_target_build(tp, tn, leaf_size, main)
        main.wait_stream(side)
        sp.record_stream(main)
        P0.record_stream(main)
        res, _ = cil_icp_run(tgt, sp, P0, prm, want_log=False, stream=main)
        out = decode_result(res)
    tgt.free(main)
    return out
