"""Target build + source-order (run of 1 iteration) timings on C4 for the libcil.so first on the path."""
import os, sys
sys.path.append(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
w = gen.c4_lidar("point_to_plane")
tg, nr = d(w.target), d(w.target_normals)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
def timed(f, reps=7):
    f(); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))
b = timed(lambda: cil.cil_target_build(tg, nr).free())
print(os.path.dirname(os.path.dirname(cil.__file__))[-20:], f"build {b:.3f} ms")
