"""C4 run time vs certificate skin parameters (min_frac, max_frac, kappa)."""
import os, sys, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
metric = sys.argv[1] if len(sys.argv) > 1 else "point_to_plane"
w = gen.c4_lidar(metric)
t = cil.cil_target_build(d(w.target), d(w.target_normals))
src, P0 = d(w.source), d(np.eye(4))
prm = cil.make_params(metric, w.max_iters, w.max_dist)
ws = cil.alloc_workspace(w.m, prm)
res = torch.zeros(256, dtype=torch.uint8, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ref = None
for mn, mx, ka in [(0.001, 0.005, 16), (0.001, 0.01, 16), (0.001, 0.02, 16), (0.001, 0.01, 32), (0.002, 0.02, 32),
                   (0.001, 0.04, 32), (0.0005, 0.005, 16), (0.001, 0.005, 8), (0.002, 0.01, 24), (0.001, 0.0075, 16)]:
    cil.set_cert_skin(mn, mx, ka)
    f = lambda: cil.cil_icp_run(t, src, P0, prm, ws=ws, res=res[:200], want_log=False)
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    r = cil.decode_result(res[:200])
    if ref is None:
        ref = r.pose
    print(f"skin min {mn} max {mx} kappa {ka}: run {np.median(ts):.3f} ms  searches/pt {cil.run_searched(ws) / w.m:.2f}"
          f"  same pose {np.array_equal(r.pose, ref)}", flush=True)
cil.set_cert_skin()
