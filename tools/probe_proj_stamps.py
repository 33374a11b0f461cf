"""Phase timeline of the persistent projective loop (CTA 0, %globaltimer): accumulate+partial,
grid barrier, partial sum, solve -- microseconds per iteration (median)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
w = gen.c3_depth()
K = cil.make_intrinsics(gen.W, gen.H, gen.FX, gen.FY, gen.CX, gen.CY)
tg = d(w.target)
t3 = cil.cil_target_build(tg, None)
n3, _ = cil.cil_estimate_normals(t3, 10, (0.0, 0.0, 0.0))
for m in (1000, 307200):
    prm = cil.make_params("point_to_plane", 30, w.max_dist)
    src = d(w.source[:m])
    for rep in range(2):
        st = torch.full((30, 8), -1, dtype=torch.int64, device="cuda")
        cil.debug_timestamps(st)
        cil.cil_proj_run(tg, n3, K, src, d(np.eye(4)), prm, want_log=False)
        torch.cuda.synchronize()
        cil.debug_timestamps(None)
    s = st.cpu().numpy().astype(np.float64) / 1e3
    ph = np.diff(s[:, :5], axis=1)
    it = np.diff(s[:, 0])
    print(f"m={m}: accumulate+partial {np.median(ph[1:, 0]):.2f} barrier {np.median(ph[1:, 1]):.2f} "
          f"sum {np.median(ph[1:, 2]):.2f} solve {np.median(ph[1:, 3]):.2f} | iteration {np.median(it):.2f} us")
