"""(Needs a trace build: tools/variants.sh trace "-DCIL_TRACE=1", then PYTHONPATH=tools/ubench/var_trace.)
Engine trace statistics on C5 (GPU box): per-query packet phases of the stateless iterate at
the identity for 2^20 and 2^22 points (cold hints)."""
import sys, os
sys.path.append(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))   # (a variant on PYTHONPATH wins)
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
f32 = lambda a: np.asarray(a, np.int32).view(np.float32)
q = lambda x: np.percentile(x, [50, 90, 99]).round(4).tolist()
for logn in [int(x) for x in (sys.argv[1:] or ["20", "22"])]:
    w = gen.c5_patches(logn)
    t = cil.cil_target_build(d(w.target), d(w.target_normals))
    src = d(w.source)
    prm = cil.make_params("point_to_plane", 1, w.max_dist)
    tr = torch.zeros(w.m * 16, dtype=torch.int32, device="cuda")
    cil.lib().cil_debug_engine_trace(tr.data_ptr())
    cil.cil_icp_iterate(t, src, d(np.eye(4)), prm, want_sys=False)
    torch.cuda.synchronize()
    cil.lib().cil_debug_engine_trace(None)
    a = tr.cpu().numpy().reshape(-1, 16)
    fl = a[:, 0]
    lane0 = np.arange(len(a)) % 32 == 0
    r0, rf = f32(a[:, 5]), f32(a[:, 7])
    found = np.isfinite(rf) & (rf < w.max_dist ** 2 * 1.0001)
    print(f"C5 2^{logn}: normal {(fl & 1).mean():.3f} outlier {((fl >> 1) & 1).mean():.3f} overflow {((fl >> 2) & 1).mean():.3f} "
          f"sparse {((fl >> 3) & 1).mean():.3f} found {found.mean():.3f}")
    print(f"   nF/packet p50/90/99 {q(a[lane0, 4])} items/query mean {a[:, 6].mean():.2f} p50/90/99 {q(a[:, 6])}")
    print(f"   radius after A p50/90/99 {q(f32(a[:, 1]))}  true d (found) p50/90/99 {q(np.sqrt(rf[found]))}")
    ck = a[lane0, 8:13].astype(np.float64)
    tot = ck.sum(0)
    print(f"   clock share A,B,C,DE,F {(tot / tot.sum()).round(3).tolist()} mean clocks/packet {tot.sum() / lane0.sum():.0f}")
    del t, src, tr
