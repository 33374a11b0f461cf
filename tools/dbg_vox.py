import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch, oracle
from tests import workloads as W
import paper_1807_00399_b200 as cil
w = W.c4("point_to_plane", rings=16, az=8000)
h = float(sys.argv[1]) if len(sys.argv) > 1 else 0.05
op, on, ok = oracle.voxel_downsample(w.target, h)
gp, _ = cil.cil_voxel_downsample(torch.as_tensor(w.target).cuda(), h)
gp = gp.cpu().numpy()
print(op.shape, gp.shape)
P = w.target.astype(np.float64)
K = np.floor(P / h).astype(np.int64)
print("key range", K.min(0), K.max(0), "span", K.max(0) - K.min(0))
# first mismatch
m = min(len(op), len(gp))
bad = np.flatnonzero(np.any(op[:m] != gp[:m], 1))
print("first mismatch rows", bad[:5])
if len(bad):
    i = bad[0]
    print("oracle", op[i-1:i+2], ok[i-1:i+2], "gpu", gp[i-1:i+2])
    print("gpu keys", np.floor(gp[i-1:i+2].astype(np.float64) / h))
# per-point keys: oracle fp64 vs a numpy recomputation, look for points whose quotient is within 1e-12 of an integer
Q = P / h
near = np.abs(Q - np.round(Q)) < 1e-9
print("points with quotient within 1e-9 of an integer:", near.sum(), P[np.any(near, 1)][:5], Q[np.any(near, 1)][:5])
if len(op) != len(gp):
    so = {tuple(np.floor(r.astype(np.float64) / h).astype(int)) for r in op}
    sg = {tuple(np.floor(r.astype(np.float64) / h).astype(int)) for r in gp}
    print("only gpu", list(sg - so)[:5], "only oracle", list(so - sg)[:5])
    ko = {tuple(k) for k in ok}
    print("oracle keys only (vs K)", len(ko), len({tuple(k) for k in K}))
