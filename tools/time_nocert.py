"""C4 run time with and without the certified warm start."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
w = gen.c4_lidar("point_to_plane")
t = cil.cil_target_build(d(w.target), d(w.target_normals))
src, P0 = d(w.source), d(np.eye(4))
prm = cil.make_params("point_to_plane", w.max_iters, w.max_dist)
ws = cil.alloc_workspace(w.m, prm)
res = torch.zeros(256, dtype=torch.uint8, device="cuda")
for cert in (True, False):
    cil.set_certificates(cert)
    f = lambda: cil.cil_icp_run(t, src, P0, prm, ws=ws, res=res[:200], want_log=False)
    f(); torch.cuda.synchronize(); ts = []
    for _ in range(5):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    print(f"certificates {cert}: {np.median(ts):.3f} ms, pose {cil.decode_result(res[:200]).pose[0, 3]:.12f}")
cil.set_certificates(True)
