"""Seeded synthetic workloads for the ICP hot path (configs C1-C5 of BASELINE.json).

This module is shared by the oracle side (tests/) and the product side (bench.py).
It holds NONE of the method's arithmetic (no nearest-neighbour search, no
normal-equation accumulation, no solve, no pose update): it only draws random
numbers and renders synthetic scenes, exactly following the input recipe written
in DESIGN.md section "Input recipe" (which restates SURVEY.md section 8(d)).

Seeding: rng = np.random.default_rng(np.random.SeedSequence([base, 399, c, s]))
with base = 1807 (extra parity seeds 1808, 1809), c the config number and
s the sub-stream: 0 scene/geometry, 1 target sampling + noise, 2 source sampling
+ noise, 3 motion.  C5 appends log2(N) to streams 1 and 2.

Everything is generated in fp64 and cast to fp32 at the end; ground-truth motions
are kept in fp64 as 4x4 row-major matrices mapping SOURCE -> TARGET frame
(the convention of the pose in include/cil.h).

Rotations are made with scipy.spatial.transform.Rotation (a library routine),
not with the method's own exponential map.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy.spatial.transform import Rotation

BASE_SEED = 1807


def rng_for(c: int, s: int, *extra: int, base: int = BASE_SEED) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([base, 399, c, s, *extra]))


def _unit(v: np.ndarray) -> np.ndarray:
    return v / np.linalg.norm(v)


def _pose(R: np.ndarray, t: np.ndarray) -> np.ndarray:
    T = np.eye(4)
    T[:3, :3] = R
    T[:3, 3] = t
    return T


@dataclass
class Workload:
    """One ICP (or NN) problem instance.  Arrays are packed row-major fp32 [n,3]."""
    name: str
    target: np.ndarray                     # float32 [n,3]
    source: np.ndarray                     # float32 [m,3] (the queries for NN configs)
    target_normals: np.ndarray | None      # float32 [n,3] or None
    gt_pose: np.ndarray | None             # float64 [4,4] source->target, None for NN configs
    metric: str = "point_to_plane"         # "point_to_plane" | "point_to_point" | "nn"
    max_dist: float = math.inf
    max_iters: int = 1
    extra: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.target.shape[0])

    @property
    def m(self) -> int:
        return int(self.source.shape[0])


# --------------------------------------------------------------------------- C1
def c1_sphere(n: int = 4096, base: int = BASE_SEED) -> Workload:
    """BASELINE.json configs[0]: 4,096 points uniform on the unit sphere, analytic
    normals; source = target rotated 5 deg about a random unit axis + translation of
    norm 0.02, plus iid N(0, 0.001^2); max dist 0.1, 20 iterations."""
    r1, r2, r3 = rng_for(1, 1, base=base), rng_for(1, 2, base=base), rng_for(1, 3, base=base)
    g = r1.standard_normal((n, 3))
    X = g / np.linalg.norm(g, axis=1, keepdims=True)
    nrm = X.copy()
    axis = _unit(r3.standard_normal(3))
    Rm = Rotation.from_rotvec(math.radians(5.0) * axis).as_matrix()
    tm = 0.02 * _unit(r3.standard_normal(3))
    Y = X @ Rm.T + tm + r2.normal(0.0, 0.001, (n, 3))
    gt = _pose(Rm.T, -Rm.T @ tm)
    return Workload("C1_sphere", X.astype(np.float32), Y.astype(np.float32),
                    nrm.astype(np.float32), gt, "point_to_plane", 0.1, 20)


# --------------------------------------------------------------------------- C2
def c2_uniform(n: int = 1 << 20, m: int = 1 << 20, base: int = BASE_SEED) -> Workload:
    """BASELINE.json configs[1]: exact 1-NN, n targets and m queries iid U[0,1)^3."""
    T = rng_for(2, 1, base=base).random((n, 3))
    Q = rng_for(2, 2, base=base).random((m, 3))
    return Workload("C2_uniform_nn", T.astype(np.float32), Q.astype(np.float32), None, None, "nn")


# --------------------------------------------------------------------------- C3
FX = FY = 525.0
CX, CY = 319.5, 239.5
W, H = 640, 480


def _tilt(rng, n0, max_deg=5.0):
    axis = _unit(rng.standard_normal(3))
    ang = math.radians(rng.uniform(0.0, max_deg))
    return Rotation.from_rotvec(ang * axis).apply(n0)


def _c3_scene(rng):
    planes = []
    for p0, n0 in (((0.0, 0.0, 3.5), (0.0, 0.0, -1.0)),   # back wall
                   ((0.0, 1.0, 0.0), (0.0, -1.0, 0.0)),   # floor (y down)
                   ((-1.5, 0.0, 0.0), (1.0, 0.0, 0.0))):  # side wall
        n = _unit(_tilt(rng, np.array(n0)))
        planes.append((np.array(p0), n))
    spheres = []
    while len(spheres) < 5:
        r = rng.uniform(0.1, 0.4)
        u = rng.uniform(60.0, W - 1 - 60.0)
        v = rng.uniform(60.0, H - 1 - 60.0)
        z = rng.uniform(0.5 + r, 3.0)
        c = z * np.array([(u - CX) / FX, (v - CY) / FY, 1.0])
        # in front of the walls and above the floor: signed distance on the camera side > r
        if all(np.dot(n, c - p0) > r for p0, n in planes):
            spheres.append((c, r))
    return planes, spheres


def _render_depth(planes, spheres, origin, R):
    """Ray-cast every pixel; rays origin + lam * (R d), d=((u-cx)/fx,(v-cy)/fy,1).
    Returns lam (== depth in the camera frame) [H*W] row-major, inf where no hit."""
    u, v = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64))
    d = np.stack([(u - CX) / FX, (v - CY) / FY, np.ones_like(u)], -1).reshape(-1, 3)
    dw = d @ R.T
    lam = np.full(d.shape[0], np.inf)
    for p0, n in planes:
        den = dw @ n
        with np.errstate(divide="ignore", invalid="ignore"):
            t = np.dot(n, p0 - origin) / den
        t = np.where(t > 0, t, np.inf)
        lam = np.minimum(lam, t)
    for c, r in spheres:
        oc = origin - c
        a = np.einsum("ij,ij->i", dw, dw)
        b = 2.0 * (dw @ oc)
        cc = oc @ oc - r * r
        disc = b * b - 4 * a * cc
        ok = disc >= 0
        sq = np.sqrt(np.where(ok, disc, 0.0))
        t1 = (-b - sq) / (2 * a)
        t2 = (-b + sq) / (2 * a)
        t = np.where(t1 > 0, t1, np.where(t2 > 0, t2, np.inf))
        lam = np.minimum(lam, np.where(ok, t, np.inf))
    return d, lam


def c3_depth(base: int = BASE_SEED) -> Workload:
    """BASELINE.json configs[2]: 640x480 organised depth frame of 3 planes + 5 spheres,
    back-projected with fx=fy=525, cx=319.5, cy=239.5, depth noise sigma=0.002 z^2;
    source = the scene re-rendered after a 3 deg / 0.03 m camera motion.
    Target normals are NOT produced here: the config asks for oracle PCA normals over
    10-NN, which tests/ attach with oracle.pca_normals (see tests/workloads.py)."""
    planes, spheres = _c3_scene(rng_for(3, 0, base=base))
    r3 = rng_for(3, 3, base=base)
    axis = _unit(r3.standard_normal(3))
    Rm = Rotation.from_rotvec(math.radians(3.0) * axis).as_matrix()
    tm = 0.03 * _unit(r3.standard_normal(3))
    out = []
    for s, (o, R) in ((1, (np.zeros(3), np.eye(3))), (2, (tm, Rm))):
        d, lam = _render_depth(planes, spheres, o, R)
        assert np.all(np.isfinite(lam)), "C3: every pixel must hit the back wall"
        z = lam + rng_for(3, s, base=base).standard_normal(lam.shape[0]) * (0.002 * lam * lam)
        out.append(z[:, None] * d)
    gt = _pose(Rm, tm)
    return Workload("C3_depth", out[0].astype(np.float32), out[1].astype(np.float32), None, gt,
                    "point_to_plane", 0.05, 30, extra={"width": W, "height": H})


# --------------------------------------------------------------------------- C4
RINGS, AZ = 64, 31250
MAX_RANGE = 80.0
GROUND_Z = -1.7


def _c4_boxes(rng, sensors, nbox=200):
    boxes = []
    while len(boxes) < nbox:
        sx, sy, sz = rng.uniform(1.0, 5.0, 3)
        rad = MAX_RANGE * math.sqrt(rng.uniform())
        ang = rng.uniform(0.0, 2 * math.pi)
        cx, cy = rad * math.cos(ang), rad * math.sin(ang)
        lo = np.array([cx - sx / 2, cy - sy / 2, GROUND_Z])
        hi = np.array([cx + sx / 2, cy + sy / 2, GROUND_Z + sz])
        ok = True
        for p in sensors:   # footprint (2-D rectangle) distance to the sensor position
            dx = max(lo[0] - p[0], 0.0, p[0] - hi[0])
            dy = max(lo[1] - p[1], 0.0, p[1] - hi[1])
            if math.hypot(dx, dy) < 2.0:
                ok = False
        if ok:
            boxes.append((lo, hi))
    return boxes


def _c4_dirs(rings=RINGS, az=AZ):
    th = np.radians(-25.0 + 28.0 * np.arange(rings) / (rings - 1))
    ph = 2 * np.pi * np.arange(az) / az
    ct, st = np.cos(th)[:, None], np.sin(th)[:, None]
    d = np.stack([ct * np.cos(ph)[None, :], ct * np.sin(ph)[None, :],
                  np.broadcast_to(st, (rings, az))], -1)
    return d.reshape(-1, 3), ph


def _c4_cast(boxes, origin, yaw, rings=RINGS, az=AZ):
    """Ray-cast the LiDAR from `origin` with heading `yaw` (about +z).
    Returns (range [R*A], normal [R*A,3], sensor-frame dirs [R*A,3]), range=inf on miss."""
    d, ph = _c4_dirs(rings, az)
    Rz = Rotation.from_rotvec([0.0, 0.0, yaw]).as_matrix()
    dw = d @ Rz.T
    rng_ = np.full(d.shape[0], np.inf)
    nrm = np.zeros_like(d)
    # ground plane z = GROUND_Z
    with np.errstate(divide="ignore", invalid="ignore"):
        tg = (GROUND_Z - origin[2]) / dw[:, 2]
    hit = (dw[:, 2] < 0) & (tg > 0)
    rng_[hit] = tg[hit]
    nrm[hit] = (0.0, 0.0, 1.0)
    world_ph = ph + yaw
    for lo, hi in boxes:
        cs = np.array([[lo[0], lo[1]], [lo[0], hi[1]], [hi[0], lo[1]], [hi[0], hi[1]]]) - origin[:2]
        ca = np.arctan2(cs[:, 1], cs[:, 0])
        cen = math.atan2((lo[1] + hi[1]) / 2 - origin[1], (lo[0] + hi[0]) / 2 - origin[0])
        rel = (ca - cen + np.pi) % (2 * np.pi) - np.pi
        a0, a1 = rel.min() - 1e-3, rel.max() + 1e-3
        relp = (world_ph - cen + np.pi) % (2 * np.pi) - np.pi
        cols = np.nonzero((relp >= a0) & (relp <= a1))[0]
        if cols.size == 0:
            continue
        idx = (np.arange(rings)[:, None] * az + cols[None, :]).reshape(-1)
        dd = dw[idx]
        with np.errstate(divide="ignore", invalid="ignore"):
            inv = 1.0 / dd
            t1 = (lo - origin) * inv
            t2 = (hi - origin) * inv
        tmin = np.minimum(t1, t2)
        tmax = np.maximum(t1, t2)
        tmin = np.where(np.isnan(tmin), -np.inf, tmin)
        tmax = np.where(np.isnan(tmax), np.inf, tmax)
        tn = tmin.max(1)
        tf = tmax.min(1)
        ax = tmin.argmax(1)
        ok = (tn <= tf) & (tn > 0) & (tn < rng_[idx])
        sel = idx[ok]
        rng_[sel] = tn[ok]
        n = np.zeros((sel.size, 3))
        n[np.arange(sel.size), ax[ok]] = -np.sign(dd[ok, ax[ok]])
        nrm[sel] = n @ Rz  # world normal -> sensor frame (R^T n)
    return rng_, nrm, d


def c4_lidar(metric: str = "point_to_plane", rings: int = RINGS, az: int = AZ,
             base: int = BASE_SEED) -> Workload:
    """BASELINE.json configs[3]: 64 rings x 31,250 azimuths, elevation -25..+3 deg, ground
    plane z=-1.7 + 200 axis-aligned boxes (sides 1-5 m) within 80 m, range noise 0.02 m,
    returns beyond 80 m dropped; source = scan after 1.5 deg yaw + 0.5 m forward motion;
    max dist 1.0 m, 50 iterations.  Normals are the analytic normals of the hit primitive
    (reading R13).  `rings`/`az` may be reduced for oracle-sized parity cases."""
    yaw = math.radians(1.5)
    t_move = np.array([0.5, 0.0, 0.0])
    boxes = _c4_boxes(rng_for(4, 0, base=base), [np.zeros(2), t_move[:2]])
    out = []
    for s, (o, y) in ((1, (np.zeros(3), 0.0)), (2, (t_move, yaw))):
        rho, nrm, d = _c4_cast(boxes, o, y, rings, az)
        noise = rng_for(4, s, base=base).normal(0.0, 0.02, rho.shape[0])
        keep = np.isfinite(rho) & (rho <= MAX_RANGE)
        pts = (rho[keep] + noise[keep])[:, None] * d[keep]
        out.append((pts, nrm[keep]))
    gt = _pose(Rotation.from_rotvec([0.0, 0.0, yaw]).as_matrix(), t_move)
    return Workload(f"C4_lidar_{metric}", out[0][0].astype(np.float32), out[1][0].astype(np.float32),
                    out[0][1].astype(np.float32), gt, metric, 1.0, 50,
                    extra={"rings": rings, "az": az})


# --------------------------------------------------------------------------- C5
def c5_patches(logn: int, base: int = BASE_SEED) -> Workload:
    """BASELINE.json configs[4]: N = 2^logn points on a union of 100 random 1x1 planar
    patches in [-5,5]^3, noise N(0, 0.005^2 I3), analytic normals; source an independent
    sample moved by 2 deg (random axis) / 0.05 about the origin; 1 point-to-plane
    iteration from identity, max dist 0.2."""
    n = 1 << logn
    r0 = rng_for(5, 0, base=base)
    cen = r0.uniform(-5.0, 5.0, (100, 3))
    Q = Rotation.random(100, random_state=r0).as_matrix()
    counts = np.full(100, n // 100)
    counts[: n % 100] += 1
    pid = np.repeat(np.arange(100), counts)

    def sample(rr):
        uv = rr.uniform(-0.5, 0.5, (n, 2))
        P = cen[pid] + uv[:, :1] * Q[pid, :, 0] + uv[:, 1:] * Q[pid, :, 1]
        return P + rr.normal(0.0, 0.005, (n, 3))

    X = sample(rng_for(5, 1, logn, base=base))
    Ys = sample(rng_for(5, 2, logn, base=base))
    r3 = rng_for(5, 3, base=base)
    Rm = Rotation.from_rotvec(math.radians(2.0) * _unit(r3.standard_normal(3))).as_matrix()
    tm = 0.05 * _unit(r3.standard_normal(3))
    Y = Ys @ Rm.T + tm
    gt = _pose(Rm.T, -Rm.T @ tm)
    return Workload(f"C5_patches_2^{logn}", X.astype(np.float32), Y.astype(np.float32),
                    Q[pid, :, 2].astype(np.float32), gt, "point_to_plane", 0.2, 1)


def by_name(name: str, **kw) -> Workload:
    table = {"c1": c1_sphere, "c2": c2_uniform, "c3": c3_depth, "c4": c4_lidar, "c5": c5_patches}
    return table[name](**kw)
