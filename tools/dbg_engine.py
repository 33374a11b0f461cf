"""Debug: NN engine (through cil_icp_iterate, identity pose, unbounded) vs brute force on
small Gaussian clouds; prints the engine trace of failing queries."""
import sys, os, time, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1807_00399_b200 as cil
from scipy.spatial.distance import cdist

f32 = lambda i: np.array([i], np.int32).view(np.float32)[0]
import itertools
modes = [int(x) for x in sys.argv[1].split(',')] if len(sys.argv) > 1 else [1, 0]
sizes = [(1000, 1000, 16), (1000, 1000, 8), (4097, 3001, 32)] if len(sys.argv) <= 2 else [(65537, 20000, 8)]
for mode, (n, m, leaf) in itertools.product(modes, sizes):
    cil.lib().cil_debug_set_flags(mode << 1)
    rng = np.random.default_rng(n + m)
    T = rng.standard_normal((n, 3)).astype(np.float32)
    Q = (rng.standard_normal((m, 3)) * 1.1).astype(np.float32)
    t = cil.cil_target_build(torch.as_tensor(T).cuda(), None, leaf_size=leaf)
    tr = torch.full((m * 16,), -7, dtype=torch.int32, device="cuda")
    cil.lib().cil_debug_engine_trace(tr.data_ptr())
    prm = cil.make_params("point_to_point", 1, math.inf)
    t0 = time.time()
    _, _, gi, gd = cil.cil_icp_iterate(t, torch.as_tensor(Q).cuda(), torch.eye(4, dtype=torch.float64, device="cuda"), prm, want_corr=True)
    torch.cuda.synchronize()
    cil.lib().cil_debug_engine_trace(None)
    gi, gd, tr = gi.cpu().numpy(), gd.cpu().numpy(), tr.cpu().numpy().reshape(m, 16)
    D = cdist(Q.astype(np.float64), T.astype(np.float64), "sqeuclidean")
    ref = np.argmin(D, 1)
    bad = np.nonzero(gi != ref)[0]
    print("mode", mode, n, m, leaf, "bad", len(bad), "time", round(time.time() - t0, 3), "flags hist", np.bincount(tr[:, 0] & 7, minlength=8), flush=True)
    for q in bad[:3]:
        r = tr[q]
        print("  q", q, "lane", q % 32, "gpu", gi[q], gd[q], "ref", ref[q], round(D[q, ref[q]], 6), "| flags", r[0], "r", f32(r[1]),
              "i0,i1", r[2], r[3], "nF", r[4], "bestD", f32(r[5]), "hint", r[6], "final", f32(r[7]), flush=True)
