"""Run time of cil_icp_run on C3 / C4 with the device's order choice (flags 0), the caller's
order (16) and the Morton order (32)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def bench(name, w, nrm):
    t = cil.cil_target_build(d(w.target), nrm)
    src, P0 = d(w.source), d(np.eye(4))
    prm = cil.make_params("point_to_plane", w.max_iters, w.max_dist)
    ws = cil.alloc_workspace(w.m, prm)
    res = torch.zeros(256, dtype=torch.uint8, device="cuda")
    for fl in (0, 16, 32):
        cil.lib().cil_debug_set_flags(fl)
        f = lambda: cil.cil_icp_run(t, src, P0, prm, ws=ws, res=res[:200], want_log=False)
        f(); torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); f(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
        print(f"{name} flags {fl}: {np.median(ts):.3f} ms, searches/pt {cil.run_searched(ws) / w.m:.2f}", flush=True)
    cil.lib().cil_debug_set_flags(0)


w3 = gen.c3_depth()
t3 = cil.cil_target_build(d(w3.target), None)
n3, _ = cil.cil_estimate_normals(t3, 10, (0.0, 0.0, 0.0))
bench("C3", w3, n3)
w4 = gen.c4_lidar("point_to_plane")
bench("C4", w4, d(w4.target_normals))
w1 = gen.c1_sphere()
bench("C1", w1, d(w1.target_normals))
