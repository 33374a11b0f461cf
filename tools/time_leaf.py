"""Leaf size 8 vs 16 on every config (run / iterate / query times)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(f, reps=5):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


P0 = d(np.eye(4))
for B in (8, 16):
    out = []
    w1 = gen.c1_sphere(); t = cil.cil_target_build(d(w1.target), d(w1.target_normals), B)
    p = cil.make_params("point_to_plane", w1.max_iters, w1.max_dist); s = d(w1.source)
    out.append(("C1 run", timed(lambda: cil.cil_icp_run(t, s, P0, p, want_log=False))))
    w2 = gen.c2_uniform(); t = cil.cil_target_build(d(w2.target), None, B); q = d(w2.source)
    out.append(("C2 query", timed(lambda: cil.cil_nn_query(t, q))))
    w3 = gen.c3_depth(); t0 = cil.cil_target_build(d(w3.target), None); n3, _ = cil.cil_estimate_normals(t0, 10, (0, 0, 0))
    t = cil.cil_target_build(d(w3.target), n3, B); p = cil.make_params("point_to_plane", w3.max_iters, w3.max_dist); s = d(w3.source)
    out.append(("C3 run", timed(lambda: cil.cil_icp_run(t, s, P0, p, want_log=False))))
    for logn in (20, 22):
        w5 = gen.c5_patches(logn); t = cil.cil_target_build(d(w5.target), d(w5.target_normals), B)
        p = cil.make_params("point_to_plane", 1, w5.max_dist); s = d(w5.source)
        out.append((f"C5 2^{logn}", timed(lambda: cil.cil_icp_iterate(t, s, P0, p, want_sys=False))))
    print(f"B={B}: " + "  ".join(f"{k} {v:.3f} ms" for k, v in out), flush=True)
