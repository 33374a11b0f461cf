"""Every BASELINE.json config on one GPU (the bench.py contract covers C4 point-to-plane;
this reports the rest): device time with CUDA events on the stream, inputs resident in HBM,
L2 flushed before every repetition; algorithmic bytes per SURVEY.md 8(d) against the measured
HBM peak.  C3 uses the library's own 10-NN PCA normals (cil_estimate_normals, timed apart).
Usage: python tools/bench_all.py [reps] > out.jsonl"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

REPS = int(sys.argv[1]) if len(sys.argv) > 1 else 5
PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists("MEASURED_PEAKS.json") else 6650.0
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


def run_cfg(name, w, metric, iters, normals=None, extra=None):
    nrm = normals if normals is not None else (d(w.target_normals) if w.target_normals is not None else None)
    t = cil.cil_target_build(d(w.target), nrm)
    src, P0 = d(w.source), d(np.eye(4))
    prm = cil.make_params(metric, iters, w.max_dist)
    ws = cil.alloc_workspace(w.m, prm)
    res = torch.zeros(256, dtype=torch.uint8, device="cuda")
    ms = timed(lambda: cil.cil_icp_run(t, src, P0, prm, ws=ws, res=res[:200], want_log=False))
    r = cil.decode_result(res[:200])
    bpp = 24 if metric == "point_to_point" else 36
    it_ms = ms / iters
    emit(config=name, metric=metric, n_source=w.m, n_target=w.n, iterations=iters, run_ms=ms, ms_per_iteration=it_ms,
         pairs_per_s=w.m * iters / (ms / 1e3), hbm_frac=bpp * w.m / (it_ms * 1e-3) / 1e9 / PEAK,
         full_searches=cil.run_searched(ws) / w.m, final_rmse=r.rmse, n_corr=r.n_corr, status=r.status, **(extra or {}))
    t.free()


w1 = gen.c1_sphere()
run_cfg("C1_sphere", w1, "point_to_plane", w1.max_iters)

w2 = gen.c2_uniform()
tg2 = d(w2.target)
t2 = cil.cil_target_build(tg2, None)
q2 = d(w2.source)
ms = timed(lambda: cil.cil_nn_query(t2, q2))
emit(config="C2_uniform_nn", metric="exact 1-NN", n_query=w2.m, n_target=w2.n, ms=ms,
     queries_per_s=w2.m / (ms / 1e3), hbm_frac=32 * w2.m / (ms * 1e-3) / 1e9 / PEAK)
bms = timed(lambda: cil.cil_target_build(tg2, None).free())       # (the target already in HBM)
emit(config="C2_uniform_build", n_target=w2.n, build_ms=bms)
t2.free()
# the uniform-grid index (CIL_INDEX_GRID), the measured winner on C2
t2g = cil.cil_target_build(tg2, None, index="grid")
ms = timed(lambda: cil.cil_nn_query(t2g, q2))
emit(config="C2_uniform_nn", index="grid", metric="exact 1-NN", n_query=w2.m, n_target=w2.n, ms=ms,
     queries_per_s=w2.m / (ms / 1e3), hbm_frac=32 * w2.m / (ms * 1e-3) / 1e9 / PEAK)
bms = timed(lambda: cil.cil_target_build(tg2, None, index="grid").free())
emit(config="C2_uniform_build", index="grid", n_target=w2.n, build_ms=bms)
t2g.free()

w3 = gen.c3_depth()
t3 = cil.cil_target_build(d(w3.target), None)
nms = timed(lambda: cil.cil_estimate_normals(t3, 10, (0.0, 0.0, 0.0)))
n3, _ = cil.cil_estimate_normals(t3, 10, (0.0, 0.0, 0.0))
emit(config="C3_depth_normals", k=10, n=w3.n, ms=nms)
run_cfg("C3_depth", w3, "point_to_plane", w3.max_iters, normals=n3, extra={"normals": "cil_estimate_normals k=10"})

# projective data association on the organised C3 frame: one
# streaming kernel per iteration; also the per-launch kernel time (no L2 flush inside a run)
K3 = cil.make_intrinsics(gen.W, gen.H, gen.FX, gen.FY, gen.CX, gen.CY)
tg3, src3, P3 = d(w3.target), d(w3.source), d(np.eye(4))
for metric in ("point_to_plane", "point_to_point"):
    prm = cil.make_params(metric, w3.max_iters, w3.max_dist)
    wsp = torch.empty(cil.cil_proj_workspace_bytes(w3.m, prm), dtype=torch.uint8, device="cuda")
    res = torch.zeros(256, dtype=torch.uint8, device="cuda")
    nrm3 = n3 if metric != "point_to_point" else None
    ms = timed(lambda: cil.cil_proj_run(tg3, nrm3, K3, src3, P3, prm, ws=wsp, res=res[:200], want_log=False))
    cil.profile_enable(True)
    cil.profile_read()
    cil.cil_proj_run(tg3, nrm3, K3, src3, P3, prm, ws=wsp, res=res[:200], want_log=False)
    st = cil.profile_read()
    cil.profile_enable(False)
    r = cil.decode_result(res[:200])
    bpp = 24 if metric == "point_to_point" else 36
    # one cooperative persistent launch runs all iterations (per-iteration launches if the grid
    # cannot be co-scheduled): per-iteration kernel time = launch time / iterations per launch
    kern_us = 1e3 * st["acc_ms"] / max(st["n_acc"], 1) / (w3.max_iters if st["n_acc"] == 1 else 1)
    emit(config="C3_depth_projective", metric=metric, n_source=w3.m, n_target=w3.n, iterations=w3.max_iters,
         run_ms=ms, ms_per_iteration=ms / w3.max_iters, pairs_per_s=w3.m * w3.max_iters / (ms / 1e3),
         hbm_frac=bpp * w3.m / (ms / w3.max_iters * 1e-3) / 1e9 / PEAK, kernel_us=kern_us,
         kernel_hbm_frac=bpp * w3.m / (kern_us * 1e-6) / 1e9 / PEAK, final_rmse=r.rmse, n_corr=r.n_corr,
         status=r.status)

# voxel-grid downsampling: the paper's 1 cm grid on C3, 5 cm on C4
w4v = gen.c4_lidar("point_to_plane")
for name, pts, h in (("C3_depth", w3.target, 0.01), ("C4_lidar", w4v.target, 0.05)):
    dp = d(pts)
    ms = timed(lambda: cil.cil_voxel_downsample(dp, h, sync=False))
    nb = cil.cil_voxel_downsample(dp, h)[0].shape[0]
    emit(config=f"{name}_voxel_downsample", bin=h, n=int(pts.shape[0]), bins=nb, ms=ms,
         points_per_s=pts.shape[0] / (ms / 1e3))
del w4v

for metric in ("point_to_plane", "point_to_point"):
    w4 = gen.c4_lidar(metric)
    run_cfg("C4_lidar", w4, metric, w4.max_iters)

for logn in (16, 18, 20, 22, 24):
    w5 = gen.c5_patches(logn)
    t5 = cil.cil_target_build(d(w5.target), d(w5.target_normals))
    src5, P0 = d(w5.source), d(np.eye(4))
    prm = cil.make_params("point_to_plane", 1, w5.max_dist)
    ws = cil.alloc_workspace(w5.m, prm)
    ms = timed(lambda: cil.cil_icp_iterate(t5, src5, P0, prm, ws=ws, want_sys=False))
    emit(config=f"C5_patches_2^{logn}", metric="point_to_plane", n=w5.m, iterate_ms=ms,
         pairs_per_s=w5.m / (ms / 1e3), hbm_frac=36 * w5.m / (ms * 1e-3) / 1e9 / PEAK)
    t5.free()
    del src5, ws
    torch.cuda.empty_cache()
