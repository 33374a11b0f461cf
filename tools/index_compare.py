"""BVH vs uniform grid (cil_index_kind), measured on the GPU box (DESIGN.md 4.1b table):
C2 cil_nn_query; C1/C3/C4/C5 stateless cil_icp_iterate at the identity (and C4 at the ground
truth); index build times.  Device time with CUDA events, L2 flushed before every repetition,
median of REPS.  Usage: python tools/index_compare.py [reps] [grid_points ...] > out.jsonl"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

REPS = int(sys.argv[1]) if len(sys.argv) > 1 else 5
GPTS = [float(x) for x in sys.argv[2:]] or [2.0]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()


def timed(fn, reps=REPS):
    fn(); fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def emit(**kw):
    print(json.dumps(kw), flush=True)


def kinds():
    yield "bvh", 0.0
    for g in GPTS:
        yield "grid", g


w2 = gen.c2_uniform()
q2 = d(w2.source)
for kind, g in kinds():
    tg = d(w2.target)
    bms = timed(lambda: cil.cil_target_build(tg, None, index=kind, grid_points=g).free())
    t2 = cil.cil_target_build(tg, None, index=kind, grid_points=g)
    ms = timed(lambda: cil.cil_nn_query(t2, q2))
    emit(config="C2_nn_query", index=kind, grid_points=g, ms=ms, queries_per_s=w2.m / (ms / 1e3), build_ms=bms)
    t2.free()


def iterate_cfg(name, w, poses):
    src = d(w.source)
    nrm = d(w.target_normals) if w.target_normals is not None else None
    prm = cil.make_params("point_to_plane" if nrm is not None else "point_to_point", 1, w.max_dist)
    ws = cil.alloc_workspace(w.m, prm)
    for kind, g in kinds():
        tg = d(w.target)
        bms = timed(lambda: cil.cil_target_build(tg, nrm, index=kind, grid_points=g).free())
        t = cil.cil_target_build(tg, nrm, index=kind, grid_points=g)
        for pn, P in poses:
            Pd = d(P)
            ms = timed(lambda: cil.cil_icp_iterate(t, src, Pd, prm, ws=ws, want_sys=False))
            emit(config=name, pose=pn, index=kind, grid_points=g, n=w.m, iterate_ms=ms, pairs_per_s=w.m / (ms / 1e3),
                 build_ms=bms)
        t.free()
    del ws
    torch.cuda.empty_cache()


w1 = gen.c1_sphere()
iterate_cfg("C1_iterate", w1, [("identity", np.eye(4))])
for logn in (16, 20, 22, 24):
    iterate_cfg(f"C5_2^{logn}_iterate", gen.c5_patches(logn), [("identity", np.eye(4))])
w4 = gen.c4_lidar("point_to_plane")
iterate_cfg("C4_iterate", w4, [("identity", np.eye(4)), ("gt", w4.gt_pose)])
