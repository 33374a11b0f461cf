"""Per-iteration time of the projective run vs source size (fixed-overhead probe)."""
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
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 30
for metric in ("point_to_plane", "point_to_point"):
    prm = cil.make_params(metric, iters, w.max_dist)
    for m in (1, 1000, 30000, 100000, 307200):
        src = d(w.source[:m])
        ws = torch.empty(cil.cil_proj_workspace_bytes(m, prm), dtype=torch.uint8, device="cuda")
        res = torch.zeros(256, dtype=torch.uint8, device="cuda")
        f = lambda: cil.cil_proj_run(tg, n3, K, src, d(np.eye(4)), prm, ws=ws, res=res[:200], want_log=False)
        f(); torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); f(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
        print(f"{metric} m={m:7d} us/iter={1e3 * np.median(ts) / iters:8.2f}")

# host enqueue cost vs device time: wall time of the (asynchronous) call, and a CUDA-graph replay
import time
prm = cil.make_params("point_to_plane", iters, w.max_dist)
for m in (1000, 307200):
    src = d(w.source[:m])
    ws = torch.empty(cil.cil_proj_workspace_bytes(m, prm), dtype=torch.uint8, device="cuda")
    res = torch.zeros(256, dtype=torch.uint8, device="cuda")
    P0 = d(np.eye(4))
    f = lambda: cil.cil_proj_run(tg, n3, K, src, P0, prm, ws=ws, res=res[:200], want_log=False)
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter(); f(); t1 = time.perf_counter(); torch.cuda.synchronize()
    print(f"m={m} host enqueue of one run: {1e6 * (t1 - t0) / iters:.2f} us/iter")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        f(); torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    print(f"m={m} graph replay us/iter={1e3 * np.median(ts) / iters:.2f}")
