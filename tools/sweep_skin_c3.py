"""C3 (depth frame, point-to-plane, 30 iterations, library 10-NN normals) run time vs the
certificate skin parameters (min_frac, max_frac, kappa; fractions of max_corr_dist)."""
import os, sys
sys.path.append(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
w = gen.c3_depth()
t0 = cil.cil_target_build(d(w.target), None)
n3, _ = cil.cil_estimate_normals(t0, 10, (0.0, 0.0, 0.0))
t = cil.cil_target_build(d(w.target), n3)
src, P0 = d(w.source), d(np.eye(4))
prm = cil.make_params("point_to_plane", w.max_iters, w.max_dist)
ws = cil.alloc_workspace(w.m, prm)
res = torch.zeros(256, dtype=torch.uint8, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
grid = [tuple(float(x) for x in g.split(",")) for g in (sys.argv[1:] or ["0.001,0.005,16"])]
for mn, mx, ka in grid:
    cil.set_cert_skin(mn, mx, ka)
    f = lambda: cil.cil_icp_run(t, src, P0, prm, ws=ws, res=res[:200], want_log=False)
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    r = cil.decode_result(res[:200])
    print(f"C3 skin ({mn},{mx},{ka}): run {np.median(ts):.3f} ms searches/pt {cil.run_searched(ws) / w.m:.2f} "
          f"pose t0 {r.pose[0, 3]:.12f}", flush=True)
