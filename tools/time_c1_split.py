"""C1 small-problem run: per-iteration cost against the source size (m = 4096 ... 32) from the
difference of a 100- and a 20-iteration cooperative launch: the m-independent part is the loop's
fixed cost (CTA partial, grid barrier, partial sum, redundant warp solve)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
I4 = d(np.eye(4))
w = gen.c1_sphere()
t = cil.cil_target_build(d(w.target), d(w.target_normals))
def timed(fn, reps=9):
    fn(); torch.cuda.synchronize(); ts=[]
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))
for m in (4096, 2048, 1024, 256, 32):
    s = d(w.source[:m])
    out = []
    for iters in (20, 100):
        prm = cil.make_params("point_to_plane", iters, w.max_dist)
        ws = cil.alloc_workspace(m, prm)
        out.append(timed(lambda: cil.cil_icp_run(t, s, I4, prm, ws=ws, want_log=False)))
    print(f"m={m}: 20 it {out[0]*1e3:.1f} us, 100 it {out[1]*1e3:.1f} us -> {(out[1]-out[0])/80*1e3:.2f} us/it, fixed {(out[0]-20*(out[1]-out[0])/80)*1e3:.1f} us", flush=True)
