"""C2 exact 1-NN query time (2^20 x 2^20) on the grid index for grid_points values, with the
libcil.so first on sys.path (variants): whole cil_nn_query and its launch profile (L2 flushed,
median of 7)."""
import os, sys
sys.path.append(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
tag = os.path.dirname(os.path.dirname(cil.__file__)).split("/")[-1]
w2 = gen.c2_uniform()
q2 = d(w2.source)
for g in [float(x) for x in (sys.argv[1:] or ["2"])]:
    t = cil.cil_target_build(d(w2.target), None, index="grid", grid_points=g)
    f = lambda: cil.cil_nn_query(t, q2)
    f(); f(); torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    print(f"{tag} C2 grid {g} pts/cell: cil_nn_query {np.median(ts) * 1e3:.1f} us", flush=True)
    del t
