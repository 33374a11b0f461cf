"""Engine trace statistics of cil_nn_query on C2 (2^20 x 2^20 uniform) + the query-sort split."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

w = gen.c2_uniform()
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
t = cil.cil_target_build(d(w.target), None)
q = d(w.source)
f32 = lambda a: np.asarray(a, np.int32).view(np.float32)
tr = torch.zeros(w.m * 16, dtype=torch.int32, device="cuda")
cil.lib().cil_debug_engine_trace(tr.data_ptr())
cil.cil_nn_query(t, q)
torch.cuda.synchronize()
cil.lib().cil_debug_engine_trace(None)
a = tr.cpu().numpy().reshape(-1, 16)
fl = a[:, 0]
lane0 = np.arange(len(a)) % 32 == 0
qq = lambda x: np.percentile(x, [50, 90, 99]).round(1).tolist()
print("normal", (fl & 1).mean().round(4), "outlier", ((fl >> 1) & 1).mean().round(4), "overflow",
      ((fl >> 2) & 1).mean().round(4), "sparse", ((fl >> 3) & 1).mean().round(4))
print("nF mean", a[lane0, 4].mean().round(1), qq(a[lane0, 4]), "items/query", a[:, 6].mean().round(2), qq(a[:, 6]),
      "r", qq(f32(a[:, 1])), "keyrange/8", qq((a[lane0, 3] - a[lane0, 2]) / 8.0)[:2])
ck = a[lane0, 8:13].astype(np.float64)
tot = ck.sum(0)
print("clock share A B C DE F:", (tot / tot.sum()).round(3).tolist(), "mean clocks/packet", round(tot.sum() / lane0.sum()))
cil.profile_enable(True); cil.profile_read()
for _ in range(5):
    cil.cil_nn_query(t, q)
torch.cuda.synchronize()
st = cil.profile_read(); cil.profile_enable(False)
print("query ms per call (incl. sort)", st["query_ms"] / max(st["n_query"], 1), "engine nn ms", st["nn_ms"] / max(st["n_nn"], 1))
