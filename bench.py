#!/usr/bin/env python
"""bench.py -- ICP point-pairs/s on B200 (BASELINE.json metric) for the north_star workload.

Default workload (N=1): BASELINE.json configs[3], the ~2M-point LiDAR scan, point-to-plane,
50 iterations, max dist 1.0 m -- the "2M-point config" the north_star target is quoted on.

A STEP is one pass of the whole hot path over one synthetic
frame pair already resident in HBM: cil_target_build (index over the target) followed by
cil_icp_run (50 fused iterations: transform, exact 1-NN, reject, J^TJ/J^Tr, on-device solve
and pose update).  value = source points x iterations / step time (pairs/s), whole job
over all ranks.  L2 is flushed (a 512 MiB device write) before every timed step.

--impl reference times the fp64 CPU oracle (oracle/, test infrastructure) on the host cores
on a bounded sample of the same workload; the driver computes the ratio itself.

Multi-GPU (torchrun, one rank per GPU): every rank aligns its own independent frame pair
(seed base 1807 + rank), no data-path collective: "scaling": "weak".
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ICP point-pairs/sec per iteration (1-NN + 6x6 reduce); % of HBM roofline"
UNIT = "point-pairs/s"


def _workload(name: str, base: int):
    import gen
    if name == "c4_plane":
        return gen.c4_lidar("point_to_plane", base=base)
    if name == "c4_point":
        return gen.c4_lidar("point_to_point", base=base)
    if name == "c1":
        return gen.c1_sphere(base=base)
    if name == "c3":
        w = gen.c3_depth(base=base)
        raise SystemExit("c3 needs oracle PCA normals; bench it through tests/ instead")
    if name.startswith("c5_"):
        return gen.c5_patches(int(name[3:]), base=base)
    raise SystemExit(f"unknown workload {name}")


def _bytes_per_pair(metric: str) -> int:
    # 12 B source + 12 B target + 12 B normal (point-to-plane) per query
    return 36 if metric == "point_to_plane" else 24


def _peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms while running."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------- our arm
def reduce_over_ranks(tot_ms: float, pairs: float, world: int, device) -> tuple[float, float]:
    """Whole-job aggregation: the timed region's duration is the MAX over ranks (device-timed
    per rank), the work is the SUM of every rank's point-pairs (each rank aligns its own
    frame pair: weak scaling, no data-path collective)."""
    if world == 1:
        return tot_ms, pairs
    import torch
    import torch.distributed as dist
    t = torch.tensor([tot_ms], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    p = torch.tensor([pairs], dtype=torch.float64, device=device)
    dist.all_reduce(p, op=dist.ReduceOp.SUM)
    dist.barrier()
    return float(t.item()), float(p.item())


def rank_seed(rank: int) -> int:
    """seed base of the frame pair rank `rank` aligns (rank 0 = BASELINE.json's configs)"""
    return 1807 + rank


def run_ours(args, rank, world, local_rank):
    import torch
    import paper_1807_00399_b200 as cil

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    w = _workload(args.workload, rank_seed(0 if args.split else rank))
    iters = args.iters or w.max_iters
    metric = w.metric
    to_dev = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(dev)
    tgt = to_dev(w.target)
    nrm = to_dev(w.target_normals) if w.target_normals is not None else None
    lo, hi = (rank * w.m // world, (rank + 1) * w.m // world) if args.split else (0, w.m)
    m_rank = hi - lo
    src = to_dev(w.source[lo:hi])
    P0 = to_dev(np.eye(4))
    prm = cil.make_params(metric, iters, w.max_dist)
    ws = cil.alloc_workspace(m_rank, prm, dev)
    res = torch.zeros(C_sizeof(cil.cil_icp_result), dtype=torch.uint8, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step(evs=None):
        t = cil.cil_target_build(tgt, nrm, args.leaf)
        if evs:
            evs[1].record(stream)
        if args.split:
            run = cil.ShardRun(t, src, P0, prm, want_log=False, ws=ws)
            for _ in range(iters):
                s = run.accumulate()
                if world > 1:
                    dist.all_reduce(s, op=dist.ReduceOp.SUM)
                run.finish()
            res.copy_(run.result())
        else:
            cil.cil_icp_run(t, src, P0, prm, ws=ws, res=res, want_log=False)
        t.free()

    if world > 1 or args.split:
        import torch.distributed as dist
    for _ in range(args.warmup):
        flush.fill_(1)
        step()
    torch.cuda.synchronize()

    # timed region: K steps, L2 flushed before each; events on the launching stream (step
    # boundaries only: per-kernel events would serialise the programmatic dependent launches)
    launches0 = cil.launch_count()
    tot_ms, build_ms, run_ms = 0.0, 0.0, 0.0
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            evs[0].record(stream)
            step(evs)
            evs[2].record(stream)
            evs[2].synchronize()
            tot_ms += evs[0].elapsed_time(evs[2])
            build_ms += evs[0].elapsed_time(evs[1])
            run_ms += evs[1].elapsed_time(evs[2])
        torch.cuda.synchronize()
    launches = cil.launch_count() - launches0
    # per-kernel launch durations for the roofline: the same K steps again with the library's
    # per-launch CUDA events on the launching stream (not part of the timed value above)
    cil.profile_read()
    cil.profile_enable(True)
    for _ in range(args.steps):
        flush.fill_(1)
        step()
    torch.cuda.synchronize()
    cil.profile_enable(False)
    prof = cil.profile_read()
    prof_iters = None
    if not args.split and not args.no_iter_profile:
        t_p = cil.cil_target_build(tgt, nrm, args.leaf)
        prof_iters = _iteration_profile(cil, t_p, src, w, metric, iters, flush, dev)
        t_p.free()
    tot_max, total_pairs = reduce_over_ranks(tot_ms, float(m_rank) * iters * args.steps, world, dev)
    r = cil.decode_result(res)
    # e2e: the public host-buffer API on every rank (pinned host inputs, H2D inside the timed
    # region, result read back to the host every step)
    e2e = _e2e(args, w, iters, cil, dev, flush, rank, world, lo, hi) if not args.no_e2e else None
    if rank != 0:
        return None
    ms_step = tot_max / args.steps
    value = total_pairs / (tot_max / 1e3)
    # dominant unit: one ICP iteration = icp_nn_kernel (correspondences) + icp_acc_kernel
    # (transform/reject/J^TJ/J^Tr/reduce/solve), each launch timed with CUDA events on the
    # launching stream inside the timed region (library profiler)
    nn_ms = prof["nn_ms"] / max(prof["n_nn"], 1)
    acc_ms = prof["acc_ms"] / max(prof["n_acc"], 1)
    sel_ms = prof["sel_ms"] / max(prof["n_sel"], 1) if prof["n_sel"] else 0.0
    it_ms = sel_ms + nn_ms + acc_ms
    bpp = _bytes_per_pair(metric)
    achieved = bpp * m_rank / (it_ms * 1e-3) / 1e9
    peak, peak_src = _peak_hbm()
    traffic = _traffic_from_profiles(args.workload, args.leaf or 16)

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if args.split else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {
            "workload": f"{w.name}: BASELINE.json configs[3] LiDAR 64x31250, {metric}, {iters} iterations, "
                        f"max dist {w.max_dist} m (target build + ICP run per step)",
            "n_target": w.n, "n_source": w.m, "iterations": iters, "leaf_size": args.leaf or 16,
            "l2": "flushed before every step (512 MiB device write)",
            "build_ms": build_ms / args.steps, "icp_ms_per_iteration": it_ms,
            "icp_select_kernel_ms": sel_ms, "icp_nn_kernel_ms": nn_ms, "icp_acc_kernel_ms": acc_ms,
            "run_ms": run_ms / args.steps,
            "full_searches_per_run": cil.run_searched(ws) / max(m_rank, 1),
            "timed_launches": {"select": prof["n_sel"], "nn": prof["n_nn"], "acc": prof["n_acc"],
                               "build": prof["n_build"]},
            "final_status": r.status, "final_n_corr": r.n_corr, "final_rmse": r.rmse,
            "parallelism": (f"one frame pair split over {world} rank(s), all-reduce of 32 fp64 per iteration"
                            if args.split else f"independent frame pair per rank x{world}"),
        },
        "roofline": {"bound": "hbm", "kernel": "icp_select_kernel+icp_nn_kernel+icp_acc_kernel (one ICP iteration, run average)",
                     "timing": "per-launch CUDA events on the launching stream over K further steps of the same workload",
                     "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "bytes_per_pair": bpp, "peak_source": peak_src,
                     "frac_of_8TBps_nominal": achieved / 8000.0},
        "roofline_issue": _issue_roofline_from_profiles(args.leaf or 16),
        "iterations_profile": prof_iters,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline and world == 1:
        out["cpu_baseline"] = _cpu_baseline(w, metric, args)
    return out


def C_sizeof(ct):
    import ctypes
    return ctypes.sizeof(ct)


def _traffic_from_profiles(workload, leaf):
    """dram bytes of one steady-state ICP iteration (select + nn + acc kernels) from the committed
    ncu --set full captures (profiles/traffic.json) -- only if they were taken with the leaf size
    the bench times (else None: the counters would describe another kernel build)"""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            t = json.load(f).get(workload)
        if t is None or int(t.get("leaf_size", -1)) != leaf:
            return None
        return t.get("steady_iteration_bytes")
    except Exception:
        return None


NCU_FULL_SEARCH = "profiles/r2_ncu_nn_it3_c4cert.txt"


def _issue_roofline_from_profiles(leaf):
    """the search kernel's instruction-issue roofline on a full-search iteration, from the
    committed ncu --set full capture: executed warp-instructions / duration against 148 SMs x 4
    schedulers x sm_max_mhz.  Refused (None) unless the capture's kernel template is the timed
    leaf size (icp_nn_kernel<leaf, 1>)."""
    import re
    p = os.path.join(ROOT, NCU_FULL_SEARCH)
    try:
        vals = {}
        lines = open(p).read().splitlines()
        m = re.search(r"icp_nn_kernel<(\d+),", lines[0])
        if not m or int(m.group(1)) != leaf:
            return None
        for line in lines:
            parts = line.split()
            if line.strip().startswith("Duration"):
                vals["us"] = float(parts[1]) * (1e-3 if parts[2] == "ns" else 1.0)
            elif line.strip().startswith("Executed Instructions"):
                vals["inst"] = float(parts[2])
            elif line.strip().startswith("Issue Slots Busy"):
                vals["busy"] = float(parts[3]) / 100.0
        mhz = 1965.0
        try:
            mhz = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"])
        except Exception:
            pass
        ach = vals["inst"] / (vals["us"] * 1e-6)
        peak = 148 * 4 * mhz * 1e6
        return {"bound": "issue", "kernel": f"icp_nn_kernel<{leaf}, 1>, full-search iteration 3 (ncu --set full capture)",
                "achieved": ach, "peak": peak, "unit": "warp-instructions/s", "frac": ach / peak,
                "ncu_issue_slots_busy": vals.get("busy"), "source": NCU_FULL_SEARCH}
    except Exception:
        return None


def _iteration_profile(cil, t, src, w, metric, iters, flush, dev):
    """SURVEY.md 8(d)'s three C4 numbers, device-timed with CUDA events (median of 5, L2 flushed
    before each): (i) a cold full-search iteration at the identity (stateless cil_icp_iterate);
    (ii) the steady certified iteration = (run(iters) - run(iters - 20)) / 20, i.e. the mean of
    the last 20 iterations of the certified run; (iii) the run average (= the headline)."""
    import torch
    P0 = torch.eye(4, dtype=torch.float64, device=dev)

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return float(np.median(ts))

    p1 = cil.make_params(metric, 1, w.max_dist)
    ws = cil.alloc_workspace(w.m, cil.make_params(metric, iters, w.max_dist), dev)
    cold = timed(lambda: cil.cil_icp_iterate(t, src, P0, p1, ws=ws, want_sys=False))
    runs = {}
    for k in (iters, max(iters - 20, 1)):
        pk = cil.make_params(metric, k, w.max_dist)
        runs[k] = timed(lambda: cil.cil_icp_run(t, src, P0, pk, ws=ws, want_log=False))
    k0 = max(iters - 20, 1)
    steady = (runs[iters] - runs[k0]) / max(iters - k0, 1)
    bpp = _bytes_per_pair(metric)
    peak, _ = _peak_hbm()
    out = {}
    for name, ms in (("i_cold_full_search_iterate", cold), ("ii_steady_certified_iteration", steady),
                     ("iii_run_average_iteration", runs[iters] / iters)):
        out[name] = {"ms": ms, "pairs_per_s": w.m / (ms * 1e-3), "hbm_frac": bpp * w.m / (ms * 1e-3) / 1e9 / peak}
    out["_how"] = ("(i) stateless cil_icp_iterate at the identity, L2 flushed; (ii) (run(%d) - run(%d)) / %d; "
                   "(iii) run(%d) / %d; target prebuilt, median of 5" % (iters, k0, iters - k0, iters, iters))
    return out


def _e2e(args, w, iters, cil, dev, flush, rank, world, lo, hi):
    """the public host-buffer path on every rank: pinned host inputs copied in, target build, the
    run (split or not), the result read back -- all inside the timed region; (max-over-ranks
    time, summed pairs) like the device-timed value"""
    import torch
    stream = torch.cuda.current_stream()
    h_t = torch.as_tensor(w.target).pin_memory()
    h_n = torch.as_tensor(w.target_normals).pin_memory() if w.target_normals is not None else None
    h_s = torch.as_tensor(np.ascontiguousarray(w.source[lo:hi])).pin_memory()
    h_res = torch.zeros(C_sizeof(cil.cil_icp_result), dtype=torch.uint8).pin_memory()
    d_t = torch.empty_like(h_t, device=dev)
    d_n = torch.empty_like(h_n, device=dev) if h_n is not None else None
    d_s = torch.empty_like(h_s, device=dev)
    P0 = torch.eye(4, dtype=torch.float64, device=dev)
    prm = cil.make_params(w.metric, iters, w.max_dist)
    ws = cil.alloc_workspace(hi - lo, prm, dev)
    res = torch.zeros(C_sizeof(cil.cil_icp_result), dtype=torch.uint8, device=dev)
    if args.split and world > 1:
        import torch.distributed as dist

    s_copy = torch.cuda.Stream(device=dev)

    def step():
        if not args.split:
            # the C-ABI host-buffer call: copies in (the source on the library's second stream,
            # overlapping the index build), build, run, result out -- all inside libcil.so
            r = cil.cil_icp_align_host(h_t, h_n, h_s, None, prm, leaf_size=args.leaf or 0)
            assert r.status == 0, r.status
            return
        # split: target + normals first on the launching stream (the build needs them), the source
        # on a second stream so that its copy overlaps the index build
        d_t.copy_(h_t, non_blocking=True)
        if d_n is not None:
            d_n.copy_(h_n, non_blocking=True)
        s_copy.wait_stream(stream)
        with torch.cuda.stream(s_copy):
            d_s.copy_(h_s, non_blocking=True)
            ev_s = torch.cuda.Event()
            ev_s.record(s_copy)
        t = cil.cil_target_build(d_t, d_n, args.leaf)
        stream.wait_event(ev_s)
        if args.split:
            run = cil.ShardRun(t, d_s, P0, prm, want_log=False, ws=ws)
            for _ in range(iters):
                sm = run.accumulate()
                if world > 1:
                    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
                run.finish()
            res.copy_(run.result())
        else:
            cil.cil_icp_run(t, d_s, P0, prm, ws=ws, res=res, want_log=False)
        h_res.copy_(res, non_blocking=True)
        t.free()

    for _ in range(max(1, args.warmup)):
        step()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(args.steps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    tmax, pairs = reduce_over_ranks(tot, float(hi - lo) * iters * args.steps, world, dev)
    h2d = h_t.numel() * 4 + (h_n.numel() * 4 if h_n is not None else 0) + h_s.numel() * 4
    return {"value": pairs / (tmax / 1e3), "unit": UNIT, "ms_per_step": tmax / args.steps,
            "h2d_bytes_per_step": int(h2d) + (0 if args.split else 128), "d2h_bytes_per_step": int(h_res.numel()),
            "call": "ShardRun (torch copies + C ABI)" if args.split else "cil_icp_align_host (C ABI, pinned host buffers)"}


# ---------------------------------------------------------------------------- oracle arm
def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def _oracle_sample(w, metric, sample_pts, iters, threads):
    """the oracle as it stands: kd-tree over the full target (timed apart), ICP on a seeded
    subset of the source (identity init, fixed iterations); threads = 0: all host cores"""
    import oracle
    all_cores = oracle.get_threads()
    oracle.set_threads(threads or all_cores)
    try:
        rng = np.random.default_rng(7)
        sel = np.sort(rng.choice(w.m, size=min(sample_pts, w.m), replace=False))
        src = np.ascontiguousarray(w.source[sel])
        t0 = time.perf_counter()
        tree = oracle.KDTree(w.target)
        t1 = time.perf_counter()
        res = oracle.icp_run(None, w.target_normals if metric != "point_to_point" else None, src, metric, iters,
                             w.max_dist, tree=tree)
        t2 = time.perf_counter()
        return {"build_s": t1 - t0, "icp_s": t2 - t1, "sample": len(sel), "pairs": len(sel) * iters,
                "cores": oracle.get_threads(), "status": res.status, "tree": tree}
    finally:
        oracle.set_threads(all_cores)


def _amortised_rate(r, w):
    """pairs/s of the sample with the index build charged in proportion to the sample's share of
    the full step (the GPU step builds once per m_full x iterations pairs)"""
    return r["pairs"] / (r["icp_s"] + r["build_s"] * r["sample"] / w.m)


def _cpu_baseline(w, metric, args):
    """the oracle on the host cores -- all cores and 1 thread, median of 3, kd-tree
    build reported apart, plus one full-source iteration at the identity (all cores)"""
    import oracle
    iters = args.iters or w.max_iters
    med = lambda rs, k: float(np.median([r[k] for r in rs]))
    allc = [_oracle_sample(w, metric, args.cpu_sample, iters, 0) for _ in range(3)]
    one = [_oracle_sample(w, metric, args.cpu_sample_1t, iters, 1) for _ in range(3)]
    tree = allc[-1]["tree"]
    full = []
    for _ in range(3):
        t0 = time.perf_counter()
        oracle.icp_system(None, w.target_normals if metric != "point_to_point" else None, w.source, np.eye(4), metric,
                          w.max_dist, tree=tree, want_corr=False)
        full.append(time.perf_counter() - t0)
    rate_all = float(np.median([_amortised_rate(r, w) for r in allc]))
    rate_one = float(np.median([_amortised_rate(r, w) for r in one]))
    return {"value": rate_all, "unit": UNIT, "cores": allc[0]["cores"], "kind": "oracle",
            "cpu_model": _cpu_model(),
            "sample": (f"{args.cpu_sample} of {w.m} source points (seeded subset) x {iters} iterations against the full "
                       f"{w.n}-point target, median of 3; the kd-tree build is timed apart and charged in proportion "
                       f"to the sample's share of a full step"),
            "all_cores": {"cores": allc[0]["cores"], "pairs_per_s": rate_all,
                          "pairs_per_s_icp_only": float(np.median([r["pairs"] / r["icp_s"] for r in allc])),
                          "kd_build_s": med(allc, "build_s"), "icp_s": med(allc, "icp_s")},
            "one_thread": {"cores": 1, "sample_points": args.cpu_sample_1t, "pairs_per_s": rate_one,
                           "pairs_per_s_icp_only": float(np.median([r["pairs"] / r["icp_s"] for r in one])),
                           "kd_build_s": med(one, "build_s"), "icp_s": med(one, "icp_s")},
            "full_source_iteration_at_identity": {"cores": allc[0]["cores"], "s": float(np.median(full)),
                                                  "pairs_per_s": w.m / float(np.median(full))}}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    w = _workload(args.workload, 1807)
    iters = args.iters or w.max_iters
    import oracle
    for _ in range(args.warmup):
        _oracle_sample(w, w.metric, max(1024, args.cpu_sample // 16), 1, 0)
    tot = 0.0
    rates = []
    for _ in range(args.steps):
        r = _oracle_sample(w, w.metric, args.cpu_sample, iters, 0)
        step = r["icp_s"] + r["build_s"] * r["sample"] / w.m
        tot += step
        rates.append(r["pairs"] / step)
    value = float(np.sum([r for r in rates]) / len(rates))
    sample = (f"{args.cpu_sample} of {w.m} source points (seeded subset) x {iters} iterations against the full "
              f"{w.n}-point target per step; the kd-tree build (timed every step) is charged in proportion to the "
              f"sample's share of the full step, as the GPU step builds once per {w.m} x {iters} pairs")
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{w.name}: BASELINE.json configs[3], {w.metric}, {iters} iterations, "
                                   f"max dist {w.max_dist} m", "n_target": w.n, "n_source": w.m},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.get_threads(), "kind": "oracle",
                             "cpu_model": _cpu_model(), "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4_plane")
    ap.add_argument("--iters", type=int, default=0, help="override the config's iteration count")
    ap.add_argument("--leaf", type=int, default=0)
    ap.add_argument("--cpu-sample", type=int, default=65536)
    ap.add_argument("--cpu-sample-1t", type=int, default=8192)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-iter-profile", action="store_true")
    ap.add_argument("--split", action="store_true",
                    help="one frame pair split across the ranks (SURVEY.md 8(e): NCCL all-reduce of the 32 "
                         "fp64 sums per iteration, strong scaling) instead of one frame pair per rank")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl")
        out = run_ours(args, rank, world, local_rank)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
