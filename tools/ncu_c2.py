"""ncu target: C2 exact 1-NN query (2^20 x 2^20), index from argv[1] (bvh | grid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil
index = sys.argv[1] if len(sys.argv) > 1 else "grid"
w = gen.c2_uniform()
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
t = cil.cil_target_build(d(w.target), None, index=index)
q = d(w.source)
for _ in range(3):
    gi, gd = cil.cil_nn_query(t, q)
torch.cuda.synchronize()
print("ok", index, int(gi[0]))
