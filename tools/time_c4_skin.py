"""C4 run time for a grid of skin parameters with the libcil.so first on sys.path (variants)."""
import os, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.append(root)
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
metric = os.environ.get("METRIC", "point_to_plane")
w = gen.c4_lidar(metric)
t = cil.cil_target_build(d(w.target), d(w.target_normals), int(os.environ.get("LEAF", "0")))
src, P0 = d(w.source), d(np.eye(4))
prm = cil.make_params(metric, w.max_iters, w.max_dist)
ws = cil.alloc_workspace(w.m, prm)
res = torch.zeros(256, dtype=torch.uint8, device="cuda")
tag = os.path.dirname(os.path.dirname(cil.__file__)).split("/")[-1]
grid = [tuple(float(x) for x in g.split(",")) for g in os.environ.get("GRID", "0.001,0.005,16").split(";")]
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
    print(f"{tag} {metric} skin ({mn},{mx},{ka}): run {np.median(ts):.3f} ms searches/pt {cil.run_searched(ws) / w.m:.2f} "
          f"pose {r.pose[0, 3]:.12f}", flush=True)
