import os, sys
sys.path.append('/root/repo')
import numpy as np, torch, gen, paper_1807_00399_b200 as cil
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
w2 = gen.c2_uniform(); tg = d(w2.target); q = d(w2.source)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
def timed(fn, reps=7):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        flush.fill_(1); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); fn(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))
for g in (1.0, 1.5, 2.0):
    b = timed(lambda: cil.cil_target_build(tg, None, index="grid", grid_points=g).free())
    t = cil.cil_target_build(tg, None, index="grid", grid_points=g)
    qq = timed(lambda: cil.cil_nn_query(t, q))
    print(f"grid_points {g}: build {b*1e3:.0f} us, query {qq*1e3:.1f} us, sum {(b+qq)*1e3:.0f} us")
