"""ncu driver: C2 exact NN (2^20 x 2^20), two queries."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil
w = gen.c2_uniform()
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
t = cil.cil_target_build(d(w.target), None, int(sys.argv[1]) if len(sys.argv) > 1 else 8)
q = d(w.source)
for _ in range(2):
    i, d2 = cil.cil_nn_query(t, q)
torch.cuda.synchronize()
print("ok", int((i >= 0).sum()))
