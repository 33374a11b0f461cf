"""Index build and source-order times (cil_target_build on C2 / C4 / C5 2^24, cil_icp_iterate on
C5 2^24 which Morton-sorts its source) with the libcil.so first on sys.path (variants)."""
import os, sys
sys.path.append(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
tag = os.path.dirname(os.path.dirname(cil.__file__)).split("/")[-1]


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


out = []
w4 = gen.c4_lidar("point_to_plane")
tg4, n4 = d(w4.target), d(w4.target_normals)
out.append(("c4_build", timed(lambda: cil.cil_target_build(tg4, n4))))
w2 = gen.c2_uniform()
tg2 = d(w2.target)
out.append(("c2_build", timed(lambda: cil.cil_target_build(tg2, None))))
w5 = gen.c5_patches(24)
tg5, n5, s5 = d(w5.target), d(w5.target_normals), d(w5.source)
out.append(("c5_24_build", timed(lambda: cil.cil_target_build(tg5, n5))))
t5 = cil.cil_target_build(tg5, n5)
p5 = cil.make_params("point_to_plane", 1, w5.max_dist); ws5 = cil.alloc_workspace(w5.m, p5)
P0 = d(np.eye(4))
out.append(("c5_24_iterate", timed(lambda: cil.cil_icp_iterate(t5, s5, P0, p5, ws=ws5, want_sys=False))))
print(tag, " ".join(f"{k} {v:.3f} ms" for k, v in out), flush=True)
