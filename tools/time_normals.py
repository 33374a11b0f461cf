"""cil_estimate_normals time on C3 (k = 10) for leaf sizes 8 and 16."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
w = gen.c3_depth()
for B in (8, 16):
    t = cil.cil_target_build(d(w.target), None, B)
    cil.cil_estimate_normals(t, 10, (0.0, 0.0, 0.0)); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); cil.cil_estimate_normals(t, 10, (0.0, 0.0, 0.0)); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    print(f"normals C3 k=10 B={B}: {np.median(ts):.3f} ms")
