"""C1 / C2 / C3 / C5 timings with the libcil.so first on sys.path (variants), to check that a
C4-tuned change does not regress the other configs."""
import os, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.append(root)
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
tag = os.path.dirname(os.path.dirname(cil.__file__)).split("/")[-1]


def timed(f, reps=5):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


out = []
w1 = gen.c1_sphere()
t1 = cil.cil_target_build(d(w1.target), d(w1.target_normals))
p1 = cil.make_params("point_to_plane", w1.max_iters, w1.max_dist)
s1, P0 = d(w1.source), d(np.eye(4))
out.append(("C1 run", timed(lambda: cil.cil_icp_run(t1, s1, P0, p1, want_log=False))))
w2 = gen.c2_uniform()
t2 = cil.cil_target_build(d(w2.target), None)
q2 = d(w2.source)
out.append(("C2 nn", timed(lambda: cil.cil_nn_query(t2, q2))))
w3 = gen.c3_depth()
t3 = cil.cil_target_build(d(w3.target), None)
n3, _ = cil.cil_estimate_normals(t3, 10, (0.0, 0.0, 0.0))
t3n = cil.cil_target_build(d(w3.target), n3)
p3 = cil.make_params("point_to_plane", w3.max_iters, w3.max_dist)
s3 = d(w3.source)
out.append(("C3 run", timed(lambda: cil.cil_icp_run(t3n, s3, P0, p3, want_log=False))))
for logn in (20, 22):
    w5 = gen.c5_patches(logn)
    t5 = cil.cil_target_build(d(w5.target), d(w5.target_normals))
    p5 = cil.make_params("point_to_plane", 1, w5.max_dist)
    s5 = d(w5.source)
    out.append((f"C5 2^{logn} iterate", timed(lambda: cil.cil_icp_iterate(t5, s5, P0, p5, want_sys=False))))
print(tag, " ".join(f"{k}: {v:.3f} ms" for k, v in out))
