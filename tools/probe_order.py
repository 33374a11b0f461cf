"""C4 run time with the source order chosen on the device vs forced caller order (flag 16)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil
for metric in ("point_to_plane",):
    w = gen.c4_lidar(metric)
    d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
    t = cil.cil_target_build(d(w.target), d(w.target_normals))
    src, P0 = d(w.source), d(np.eye(4))
    prm = cil.make_params(metric, 50, 1.0)
    ws = cil.alloc_workspace(w.m, prm)
    for fl in (0, 16, 0, 16):
        cil.lib().cil_debug_set_flags(fl)
        cil.cil_icp_run(t, src, P0, prm, ws=ws, want_log=False); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); cil.cil_icp_run(t, src, P0, prm, ws=ws, want_log=False); e1.record(); torch.cuda.synchronize()
        perm = ws[-(4 * w.m + 12 * w.m + 512):].view(torch.uint8)
        print(metric, "flags", fl, "ms", round(e0.elapsed_time(e1), 3), flush=True)
