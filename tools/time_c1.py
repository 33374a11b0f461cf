"""C1 (4,096-point sphere, 20 iterations) run and iterate timing, small path vs tree path."""
import sys, os
sys.path.append(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil
w = gen.c1_sphere()
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
for flags in (0, 64):
    cil.set_debug_flags(flags)
    t = cil.cil_target_build(d(w.target), d(w.target_normals))
    src, P0 = d(w.source), d(np.eye(4))
    prm = cil.make_params("point_to_plane", w.max_iters, w.max_dist)
    prm1 = cil.make_params("point_to_plane", 1, w.max_dist)
    ws = cil.alloc_workspace(w.m, prm)
    res = torch.zeros(256, dtype=torch.uint8, device="cuda")
    for name, fn in (("run", lambda: cil.cil_icp_run(t, src, P0, prm, ws=ws, res=res[:200], want_log=False)),
                     ("iterate", lambda: cil.cil_icp_iterate(t, src, P0, prm1, ws=ws, want_sys=False))):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); fn(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
        print(f"flags {flags} {name}: median {np.median(ts)*1e3:.1f} us", flush=True)
    r = cil.decode_result(res[:200]); print("  rmse", r.rmse, "iters", r.iterations, "status", r.status)
cil.set_debug_flags(0)
