"""Per-iteration profile of cil_icp_run on C4 (GPU box): for k = 1..K, run k iterations and
difference the cumulative kernel times and search counts; also the pose step per iteration."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

metric = sys.argv[1] if len(sys.argv) > 1 else "point_to_plane"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 50
gaps = [tuple(float(v) for v in x.split(':')) for x in sys.argv[3].split(',')] if len(sys.argv) > 3 else [(0.001, 0.005, 16.0)]
flags = [int(x) for x in sys.argv[4].split(',')] if len(sys.argv) > 4 else [0]
w = gen.c4_lidar(metric)
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
t = cil.cil_target_build(d(w.target), d(w.target_normals) if w.target_normals is not None else None, 8)
src, P0 = d(w.source), d(np.eye(4))
R = np.linalg.norm(w.source, axis=1).max()
import itertools
for gap, fl in itertools.product(gaps, flags):
    cil.set_cert_skin(*gap)
    cil.lib().cil_debug_set_flags(fl)
    prev = None
    rows = []
    for k in range(1, K + 1):
        prm = cil.make_params(metric, k, 1.0)
        ws = cil.alloc_workspace(w.m, prm)
        cil.cil_icp_run(t, src, P0, prm, ws=ws, want_log=False)
        torch.cuda.synchronize()
        cil.profile_enable(True); cil.profile_read()
        res, _ = cil.cil_icp_run(t, src, P0, prm, ws=ws, want_log=False)
        torch.cuda.synchronize()
        pr = cil.profile_read(); cil.profile_enable(False)
        cur = (pr["sel_ms"], pr["nn_ms"], pr["acc_ms"], cil.run_searched(ws), cil.decode_result(res).pose,
               cil.run_point_certified(ws))
        if prev is None:
            dsel, dnn, dacc, dsr = cur[0], cur[1], cur[2], cur[3]
            dpc = cur[5]
            step = np.nan
        else:
            dsel, dnn, dacc, dsr = (cur[i] - prev[i] for i in range(4))
            dpc = cur[5] - prev[5]
            dP = np.linalg.inv(prev[4]) @ cur[4]
            ang = np.arccos(np.clip((np.trace(dP[:3, :3]) - 1) / 2, -1, 1))
            step = ang * R + np.linalg.norm(dP[:3, 3])     # displacement bound at the max range
        rows.append((k - 1, dsel * 1e3, dnn * 1e3, dacc * 1e3, dsr / w.m, step, dpc / w.m))
        prev = cur
    print(f"gap {gap} flags {fl}: iteration | sel us | nn us | acc us | searched frac | step bound m (prev->this)")
    for r in rows:
        print(f"  {r[0]:3d} {r[1]:8.1f} {r[2]:8.1f} {r[3]:7.1f}  {r[4]:6.3f}  {r[5]:.3g}  pcert {r[6]:.3f}", flush=True)
    tot = sum(r[1] + r[2] + r[3] for r in rows)
    print(f"  TOTAL gap {gap} flags {fl}: {tot/1e3:.2f} ms (first 10: {sum(r[1]+r[2]+r[3] for r in rows[:10])/1e3:.2f}), "
          f"full-equiv {sum(r[4] for r in rows):.2f}", flush=True)
