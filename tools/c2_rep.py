import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil
w = gen.c2_uniform()
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
for leaf in (8, 16):
    t = cil.cil_target_build(d(w.target), None, leaf)
    q = d(w.source)
    ts = []
    for r in range(12):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); cil.cil_nn_query(t, q); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(leaf, [round(x, 3) for x in ts])
