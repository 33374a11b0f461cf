"""Per-iteration timeline of the ICP kernels from %globaltimer stamps (cil_debug_timestamps):
gaps between kernels, body and the last-CTA tail (reduction + solve), in microseconds."""
import os, sys
sys.path.append(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()


def show(name, st, iters):
    s = st.cpu().numpy().astype(np.float64)
    s[s < 0] = np.nan
    s = (s - np.nanmin(s)) / 1e3
    rows = []
    for it in range(iters):
        r = s[it]
        first = np.nanmin(r[:3])
        prev_end = s[it - 1, 4] if it else np.nan
        rows.append((first - prev_end, r[1] - r[0], r[2] - np.nanmax([r[0], r[1]]) if not np.all(np.isnan(r[:2])) else np.nan,
                     r[3] - r[2], r[4] - r[3]))
    a = np.array(rows)
    med = np.nanmedian(a[1:], 0) if iters > 1 else a[0]
    t = np.array([[s[it, 5] - s[it, 3], s[it, 6] - s[it, 5], s[it, 4] - s[it, 6]] for it in range(iters)])
    print(f"   tail split: reduce {np.nanmedian(t[:, 0]):.2f}  solve {np.nanmedian(t[:, 1]):.2f}  update {np.nanmedian(t[:, 2]):.2f}")
    print(f"{name}: median us  gap(prev solve->next start) {med[0]:.2f}  sel->nn {med[1]:.2f}  nn->acc {med[2]:.2f}  "
          f"acc body {med[3]:.2f}  last-CTA tail {med[4]:.2f}   total/iter {(s[iters - 1, 4] - np.nanmin(s[0, :3])) / iters:.2f}")


w = gen.c3_depth()
K = cil.make_intrinsics(gen.W, gen.H, gen.FX, gen.FY, gen.CX, gen.CY)
tg = d(w.target)
t3 = cil.cil_target_build(tg, None)
n3, _ = cil.cil_estimate_normals(t3, 10, (0.0, 0.0, 0.0))
iters = 30
for m in (1000, 307200):
    prm = cil.make_params("point_to_plane", iters, w.max_dist)
    src = d(w.source[:m])
    for rep in range(2):
        st = torch.full((iters, 8), -1, dtype=torch.int64, device="cuda")
        cil.debug_timestamps(st)
        cil.cil_proj_run(tg, n3, K, src, d(np.eye(4)), prm, want_log=False)
        torch.cuda.synchronize()
        cil.debug_timestamps(None)
    show(f"proj m={m}", st, iters)

w1 = gen.c1_sphere()
t1 = cil.cil_target_build(d(w1.target), d(w1.target_normals))
prm = cil.make_params("point_to_plane", w1.max_iters, w1.max_dist)
for rep in range(2):
    st = torch.full((w1.max_iters, 8), -1, dtype=torch.int64, device="cuda")
    cil.debug_timestamps(st)
    cil.cil_icp_run(t1, d(w1.source), d(np.eye(4)), prm, want_log=False)
    torch.cuda.synchronize()
    cil.debug_timestamps(None)
show("C1 icp_run", st, w1.max_iters)
if len(sys.argv) > 1:
    w4 = gen.c4_lidar("point_to_plane")
    t4 = cil.cil_target_build(d(w4.target), d(w4.target_normals))
    prm = cil.make_params("point_to_plane", w4.max_iters, w4.max_dist)
    for rep in range(2):
        st = torch.full((w4.max_iters, 8), -1, dtype=torch.int64, device="cuda")
        cil.debug_timestamps(st)
        cil.cil_icp_run(t4, d(w4.source), d(np.eye(4)), prm, want_log=False)
        torch.cuda.synchronize()
        cil.debug_timestamps(None)
    show("C4 icp_run", st, w4.max_iters)
    s = st.cpu().numpy().astype(np.float64); s = (s - s.min()) / 1e3
    tot = {"sel": 0.0, "nn": 0.0, "acc": 0.0, "tail": 0.0, "gap": 0.0}
    for it in range(w4.max_iters):
        r = [s[it, 1] - s[it, 0], s[it, 2] - s[it, 1], s[it, 3] - s[it, 2], s[it, 4] - s[it, 3],
             (s[it + 1, 0] - s[it, 4]) if it + 1 < w4.max_iters else 0.0]
        for k, v in zip(tot, r):
            tot[k] += v
        print(f"  C4 it {it:2d}: sel {r[0]:7.1f} nn {r[1]:7.1f} acc {r[2]:6.1f} tail {r[3]:5.1f} gap {r[4]:5.1f}")
    print("  C4 totals (ms):", {k: round(v / 1e3, 3) for k, v in tot.items()})
