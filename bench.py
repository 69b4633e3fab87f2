#!/usr/bin/env python3
"""Throughput of the fused projected dual-ascent iteration (arXiv 2406.13191)
on B200, in dual-ascent instance-iterations per second (BASELINE.json metric).

Default workload = BASELINE.json configs[4]: the 10000-bus / 12700-branch /
2500-generator network, 8192 load-scenario / line-switching instances, linear
cost, form F2.  Multi-GPU default "scaling": "strong" -- the literal configs[4]:
ONE 8192-instance batch sharded over the N GPUs (rank r takes a contiguous
shard; 1024 instances per GPU at N = 8, which the batched path covers with
split tiles: one wave of 144 CTAs); --scaling weak gives every rank its own
configs[4]-sized batch instead (rank r: instances [8192 r, 8192 (r+1)) of the
seeded sweep).

A "step" is one ascent iteration (S1-S4) over the rank's whole batch.  The
timed region is one dcopf_dual_iterate(K) call = ONE persistent kernel launch
running the K iterations plus the final evaluation at y_K (the evaluation is
not counted as work, so the reported rate is conservative).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload config4|config4b|config0|config1|config2|config3|config3q]
                  [--form F2|F1|KVL|PTDF]

--form PTDF runs the paper's dense-PTDF Eq. 1 on the dense
path (two fused fp64 DMMA GEMMs per step); it takes load-only batches, so its
workload is config4b (or a single-instance config); its roofline is the fp64
tensor-core peak measured live (cuBLAS DGEMM through torch.matmul), or HBM for
batches of <= 4 instances (matrix-vector kernels).  --decay inv:T | step:F:N
gives the paper's step decay (e.g. config 3, PTDF, --opt adam --alpha 5
--decay inv:200: the fastest time to a 1e-3 gap measured).

Multi-GPU: launched by torchrun; one process per GPU; the instances are
sharded with no communication in the loop; one NCCL all_gather of the
per-instance (bound, best, status) after the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2406_13191_b200 import instances as inst  # noqa: E402
from paper_2406_13191_b200.distributed import gather_instance_results, shard  # noqa: E402

WORKLOADS = {
    # name: (config, quadratic, batch)
    "config0": (0, False, 1),
    "config1": (1, False, 1),
    "config2": (2, True, 1),
    "config3": (3, False, 1),
    "config3q": (3, True, 1),
    "config4": (4, False, inst.CONFIG4_BATCH),
    "config4b": (4, False, inst.CONFIG4_BATCH),
}
METRIC = "dual-ascent instance-iterations/sec"
# ascent-step variants: (oracle/library variant id, hyperparameters, default step)
OPTS = {
    "plain": (0, {}, 1e-3),
    "gdm": (1, {"rho": 0.9}, 1e-3),
    "gdm_classic": (2, {"rho": 0.9}, 1e-3),
    "adagrad": (3, {"eps": 1e-8}, 1.0),
    "adam": (4, {"beta1": 0.9, "beta2": 0.999, "eps": 1e-8}, 0.1),
}


def opt_spec(args):
    v, hp, a0 = OPTS[args.opt]
    return dict(variant=v, **hp), (args.alpha if args.alpha is not None else a0)


def gap_key(args):
    _, alpha = opt_spec(args)
    return (f"{args.workload}/{args.form}" + ("" if args.opt == "plain" else f"/{args.opt}/{alpha:g}")
            + (f"/{args.decay}" if args.decay else ""))
UNIT = "instance-iterations/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="config4", choices=sorted(WORKLOADS))
    ap.add_argument("--form", default="F2", choices=["F2", "F1", "KVL", "PTDF"],
                    help="F2 flow box (default), F1 limit rows, KVL cycle basis, PTDF dense (load-only batches)")
    ap.add_argument("--path", default="auto", choices=["auto", "batched", "single", "cluster", "dense"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gap", action="store_true", help="skip the time-to-gap run (the workload's full K)")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong (default): configs[4] split over the ranks; weak: each rank its own configs[4]-sized batch")
    ap.add_argument("--opt", default="plain", choices=sorted(OPTS),
                    help="ascent-step variant (PAPER.md:245); non-plain variants run on the cluster path")
    ap.add_argument("--alpha", type=float, default=None, help="step (default: the variant's)")
    ap.add_argument("--decay", default=None, help="step decay: inv:T (alpha/(1+k/T)) or step:F:N (alpha F^floor(k/N))")
    ap.add_argument("--tile", default=None,
                    help="V,C: batched path tiling (instances per lane, parts per tile); default: the library's choice")
    ap.add_argument("--batch", type=int, default=None,
                    help="instances of the config4/config4b sweep (default 8192 = configs[4]); e.g. 1024 = one "
                         "rank's shard of the literal 8-GPU split measured on one GPU")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 9]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def cpu_model():
    """The host CPU's model name (the cpu_baseline's hardware)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def make_inputs(workload, lo, hi, total=inst.CONFIG4_BATCH):
    config, quad, _ = WORKLOADS[workload]
    net = inst.make_network(config, quadratic=quad)
    if config == 4:
        batch = inst.config4_batch(net, range(lo, hi), variant="4b" if workload == "config4b" else "4",
                                   total=max(total, hi))
    else:
        batch = inst.single_batch(net)
    return net, batch


def fp64_peak_tflops(dev):
    """The fp64 tensor-core roofline for the PTDF form, measured here: cuBLAS
    DGEMM 8192^3 through torch.matmul, best of 5 (MEASURED_PEAKS.json has no
    fp64 entry and B200_PROFILING.md no fp64 fallback)."""
    import torch
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(2):
        a @ b
    best = None
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    del a, b
    return 2.0 * n ** 3 / (best / 1e3) / 1e12


def ptdf_oracle_rate(net, batch, cores, target_s=12.0, opt=None):
    """oracle/ptdf.py (numpy, BLAS threads = the host's cores) on a bounded
    sample: a few instances x K steps, H_a built outside the timed part."""
    from oracle import ptdf as P
    Ha = P.ptdf(net)
    n_inst = min(batch.B, 16)
    loads = batch.load[np.linspace(0, batch.B - 1, n_inst).astype(int)]
    K0 = 3
    t0 = time.perf_counter()
    P.solve(net, loads, K0, inst.alpha_schedule(K0), Ha=Ha, opt=opt)
    dt = max(time.perf_counter() - t0, 1e-6)
    K = int(max(K0, min(100000, K0 * target_s / dt)))
    t0 = time.perf_counter()
    P.solve(net, loads, K, inst.alpha_schedule(K), Ha=Ha, opt=opt)
    dt = time.perf_counter() - t0
    return n_inst * K / dt, f"{n_inst} instances x {K} iterations ({dt:.1f} s wall), numpy BLAS, H_a precomputed"


def cpu_oracle_rate(net, batch, form, cores, target_s=12.0, opt=None):
    """The oracle as it stands, timed on this host's cores over a bounded
    sample of the workload (instances x iterations), inst-it/s."""
    import oracle
    B = batch.B
    n_inst = min(B, max(1, 4 * cores)) if B > 1 else 1
    idx = np.linspace(0, B - 1, n_inst).astype(int) if B > 1 else np.array([0])
    loads = batch.load[idx]
    outs = None if batch.outages is None else batch.outages[idx]
    # calibrate the iteration count to ~target_s of wall time
    K0 = 20
    t0 = time.perf_counter()
    oracle.solve(net, loads, outages=outs, K=K0, alpha=inst.alpha_schedule(K0), form=form, threads=cores, opt=opt)
    dt = max(time.perf_counter() - t0, 1e-6)
    K = int(max(K0, min(200000, K0 * target_s / dt)))
    t0 = time.perf_counter()
    oracle.solve(net, loads, outages=outs, K=K, alpha=inst.alpha_schedule(K), form=form, threads=cores, opt=opt)
    dt = time.perf_counter() - t0
    return n_inst * K / dt, f"{n_inst} instances x {K} iterations ({dt:.1f} s wall)"


def time_to_gap(args, h, net, batch, lo, hi, load_dev, outs_dev, stream, world, dev, rel=1e-3):
    import torch
    import torch.distributed as tdist
    key = gap_key(args)
    try:
        ref = json.load(open(os.path.join(ROOT, "tests", "golden", "targets.json")))[key]
    except (OSError, KeyError, ValueError):
        return {"unavailable": f"no oracle reference for {key} (run tools/make_targets.py)"}
    K = int(ref["K"])
    ids = np.asarray(ref["instance_ids"], dtype=np.int64)
    best_ref = np.asarray(ref["best"], dtype=np.float64)
    B = batch.B
    target = np.full(B, np.inf)
    mine = (ids >= lo) & (ids < hi)
    # within `rel` of the reference on the lower side: best >= ref - rel |ref|
    target[ids[mine] - lo] = best_ref[mine] - rel * np.abs(best_ref[mine])
    h.set_instance_batch(load_dev, outs_dev, stream=stream)
    h.set_target(target, stream=stream)
    alpha = inst.alpha_schedule(K, float(ref["alpha"]), ref.get("decay"))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    h.iterate(K, alpha, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    run_s = e0.elapsed_time(e1) / 1e3
    hit = h.get_first_hit()[ids[mine] - lo] if mine.any() else np.zeros(0, np.int64)
    reached = int(np.sum(hit >= 0))
    worst = int(hit.max()) if reached == len(hit) and len(hit) else -1
    secs = run_s * worst / K if worst >= 0 else None
    t = torch.tensor([run_s, secs if secs is not None else -1.0, reached, len(hit)], dtype=torch.float64, device=dev)
    if world > 1:
        tmax = t.clone()
        tdist.all_reduce(tmax, op=tdist.ReduceOp.MAX)
        tsum = t.clone()
        tdist.all_reduce(tsum, op=tdist.ReduceOp.SUM)
        run_s, reached, n = float(tmax[0]), int(tsum[2]), int(tsum[3])
        secs = float(tmax[1]) if reached == n and n else None
    else:
        n = len(hit)
    degenerate = bool(np.all(best_ref[mine] == 0.0))
    out = {"rel_gap": rel, "K": K, "alpha": ref["alpha"], "reference": "oracle final running best at the same K "
           "and schedule (tests/golden/targets.json)", "sampled_instances": n, "reached": reached,
           "max_hit_iteration": worst if world == 1 else None, "seconds": None if degenerate else secs,
           "run_seconds_full_K": run_s, "reference_best_range": [float(best_ref.min()), float(best_ref.max())],
           "degenerate": degenerate}
    if degenerate:
        out["note"] = ("degenerate reference: the oracle's best bound after K steps is g(y_0) = 0 (this form and step "
                       "never rise above the starting bound here, DESIGN.md §6b), so there is no time to report")
    popt = ref.get("primal_opt")
    if popt is not None and mine.any():  # (ii): the true gap of the GPU's best bound after K, vs the optimum
        best = np.empty(batch.B)
        h.get_bound(best=best)
        po = np.atleast_1d(np.asarray(popt, dtype=np.float64))
        po = po[mine] if po.size == len(ids) else po[:1]
        b = best[ids[mine] - lo][:po.size]
        gaps = (po - b) / np.abs(po)
        out["primal_opt"] = float(po[0]) if po.size == 1 else "per sampled instance (HiGHS)"
        out["true_gap_at_K"] = float(gaps[0]) if po.size == 1 else {"median": float(np.median(gaps)),
                                                                    "max": float(np.max(gaps))}
    return out


# the batched route's step schedule: Adam with alpha_k = 48 * 0.5^floor(k/40)
# (the paper's step decay; reading A-26), chosen among 70
# schedules by tools/ptdf_batch_schedule_explore.py on the covered instances
# with ids = 0 mod 32 and confirmed on the other half (16 mod 32): 334 / 334
# iterations to the last hit (alpha_k = 5/(1+k/200), round 2's first choice:
# 3 008; profiles/r2/ptdf_sched/)
TRUE_GAP_ALPHA, TRUE_GAP_DECAY = 48.0, "step:0.5:40"


def single_true_gap(args, h, batch, load_dev, stream, rel=1e-3, chunk=250):
    """Time to a TRUE 1e-3 gap on one instance (configs 1-3): the exact
    optimum of Eq. 1 for the workload (HiGHS; Kelley cutting planes for QP,
    tests/golden/targets.json, tools/make_targets.py) as the target, the
    bench's own form / step / schedule from y_0, in chunks of `chunk` steps
    until the running best reaches it (the first hit recorded on device), at
    most the workload's K.  Reports the device time at the hit iteration (the
    chunks before it plus its chunk prorated) and the time of the chunks run."""
    import torch
    try:
        refs = json.load(open(os.path.join(ROOT, "tests", "golden", "targets.json")))
    except (OSError, ValueError):
        return {"unavailable": "no targets.json"}
    wl = args.workload + "/"
    popt = next((r["primal_opt"] for k, r in refs.items() if k.startswith(wl) and r.get("primal_opt") is not None),
                None)
    if popt is None or batch.B != 1:
        return {"unavailable": f"no exact optimum for {args.workload}"}
    popt = float(np.atleast_1d(popt)[0])
    K_max = int(inst.ITERS[WORKLOADS[args.workload][0]])
    ospec, alpha0 = opt_spec(args)
    alpha = inst.alpha_schedule(K_max, alpha0, args.decay)
    h.set_instance_batch(load_dev, None, stream=stream)  # from y_0 (resets the multipliers and the state)
    if args.opt != "plain":
        h.set_optimizer(ospec["variant"], ospec.get("rho", 0.0), ospec.get("beta1", 0.0), ospec.get("beta2", 0.0),
                        ospec.get("eps", 0.0))
    h.set_target(np.array([popt - rel * abs(popt)]), stream=stream)
    chunks, k0, hit = [], 0, -1
    while k0 < K_max:
        n = min(chunk, K_max - k0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h.iterate(n, alpha[k0:k0 + n], stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        chunks.append((k0, n, e0.elapsed_time(e1)))
        k0 += n
        hit = int(h.get_first_hit()[0])
        if hit >= 0:
            break
    best = np.empty(1)
    h.get_bound(best=best)
    at_hit = None
    if hit >= 0:
        at_hit = sum(ms for (c0, n, ms) in chunks if c0 + n <= hit)
        for (c0, n, ms) in chunks:
            if c0 <= hit < c0 + n:
                at_hit += ms * (hit - c0 + 1) / n
        at_hit /= 1e3
    return {"rel_gap": rel, "reference": "exact optimum of Eq. 1 (HiGHS; tests/golden/targets.json)",
            "primal_opt": popt, "schedule": {"alpha": alpha0, "decay": args.decay}, "hit_iteration": hit if hit >= 0
            else None, "seconds": at_hit, "seconds_run": sum(ms for (_, _, ms) in chunks) / 1e3,
            "iterations_run": k0, "true_gap_at_stop": (popt - float(best[0])) / abs(popt),
            "timing": f"device events over iterate() chunks of {chunk} steps; seconds = the chunks before the hit "
                      "+ the hit's chunk prorated"}


def batched_true_gap(dev, stream, rel=1e-3, chunk=50, K_max=5000):
    """Time to a TRUE 1e-3 gap on the batched workload (BASELINE.json metric
    "time to 1e-3 gap"; Tables 1-3 report t(s) to Gap%): the whole
    config-4b batch (8192 feasible instances) on the route that closes the gap
    fastest -- the paper's own dense-PTDF form (Eq. 1) with Adam and step decay
    (TRUE_GAP_ALPHA, TRUE_GAP_DECAY) -- until EVERY covered instance's
    running best is within 1e-3 of its exact LP optimum (HiGHS, 512 instances:
    every 16th, tests/golden/optima_config4b.json).  The kernels record each
    instance's first hit on device; the batch runs in chunks of `chunk` steps
    and stops after the chunk in which the last covered instance hit, so the
    reported seconds (device time of the chunks run) bound the true time from
    above."""
    import torch
    from paper_2406_13191_b200 import dual
    try:
        ref = json.load(open(os.path.join(ROOT, "tests", "golden", "optima_config4b.json")))
    except (OSError, ValueError):
        return {"unavailable": "no optima (run tools/make_optima.py)"}
    net, batch = make_inputs("config4b", 0, inst.CONFIG4_BATCH)
    B = batch.B
    ids = np.asarray(ref["instance_ids"], dtype=np.int64)
    popt = np.asarray(ref["primal_opt"], dtype=np.float64)
    target = np.full(B, np.inf)
    target[ids] = popt - rel * np.abs(popt)
    h = dual.DcopfDual(net, form=dual.FORM_PTDF, path=dual.PATH_DENSE, device=dev.index or 0)
    v, hp, _ = OPTS["adam"]
    h.set_optimizer(v, 0.0, hp["beta1"], hp["beta2"], hp["eps"])
    load_dev = torch.from_numpy(np.ascontiguousarray(batch.load.T)).to(dev)
    h.set_instance_batch(load_dev, None, stream=stream)
    h.set_target(target, stream=stream)
    alpha = inst.alpha_schedule(K_max, TRUE_GAP_ALPHA, TRUE_GAP_DECAY)
    total_ms, k0, hit, chunks = 0.0, 0, None, []
    while k0 < K_max:
        n = min(chunk, K_max - k0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h.iterate(n, alpha[k0:k0 + n], stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        chunks.append((k0, n, ms))
        total_ms += ms
        k0 += n
        hit = h.get_first_hit()[ids]
        if np.all(hit >= 0):
            break
    # device time until the last covered instance's hit: the chunks before
    # its chunk, plus that chunk prorated over its iterations (the reported
    # "seconds" are the chunks actually run: an upper bound)
    at_hit = None
    if np.all(hit >= 0):
        kh = int(hit.max())
        at_hit = sum(ms for (c0, n, ms) in chunks if c0 + n <= kh)
        for (c0, n, ms) in chunks:
            if c0 <= kh < c0 + n:
                at_hit += ms * (kh - c0 + 1) / n
        at_hit /= 1e3
    best = np.empty(B)
    h.get_bound(best=best)
    gaps = (popt - best[ids]) / np.abs(popt)
    h.close()
    reached = int(np.sum(hit >= 0))
    return {"route": f"config4b (8192 instances), form PTDF (dense, PAPER.md Eq. 1), Adam, alpha_k = "
                     f"{TRUE_GAP_ALPHA:g} x schedule {TRUE_GAP_DECAY}",
            "rel_gap": rel, "reference": "exact LP optimum per instance (HiGHS; tests/golden/optima_config4b.json)",
            "covered_instances": int(len(ids)), "reached": reached,
            "seconds": (total_ms / 1e3) if reached == len(ids) else None,
            "max_hit_iteration": int(hit.max()) if reached == len(ids) else None,
            "iterations_run": k0, "seconds_run": total_ms / 1e3, "seconds_at_last_hit_prorated": at_hit,
            "true_gap_at_stop": {"median": float(np.median(gaps)), "max": float(np.max(gaps))},
            "timing": f"device events over the iterate() chunks of {chunk} steps actually run (each call "
                      "ends with the evaluation at its last point)"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    form = {"F2": 0, "F1": 1, "KVL": 2, "PTDF": 3}[args.form]
    _, _, B = WORKLOADS[args.workload]
    net, batch = make_inputs(args.workload, 0, B if B == 1 else min(B, 256))
    cores = os.cpu_count() or 1
    per_step = []
    import oracle
    n_inst = min(batch.B, 2 * cores)
    loads = batch.load[:n_inst]
    outs = None if batch.outages is None else batch.outages[:n_inst]
    K_s = 50 if net.n_bus > 1000 else 2000
    a = inst.alpha_schedule(K_s)
    Ha = None
    if form == 3:
        from oracle import ptdf as P
        Ha = P.ptdf(net)
        n_inst = min(batch.B, 16)
        loads = batch.load[:n_inst]
        K_s = 5 if net.n_bus > 1000 else 2000
        a = inst.alpha_schedule(K_s)
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        if form == 3:
            P.solve(net, loads, K_s, a, Ha=Ha, opt=opt_spec(args)[0])
        else:
            oracle.solve(net, loads, outages=outs, K=K_s, alpha=a, form=form, threads=cores, opt=opt_spec(args)[0])
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            per_step.append(dt)
    T = sum(per_step)
    value = n_inst * K_s * args.steps / T
    sample = (f"{n_inst} instances x {K_s} iterations per step, "
              + ("oracle/ptdf.py numpy BLAS" if form == 3 else "oracle/dcopf_oracle.c OpenMP over instances"))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, BASELINE.json recipe)",
            "config": {"workload": args.workload, "form": args.form, "n_bus": net.n_bus,
                       "n_branch": net.n_branch, "n_gen": net.n_gen, "B": batch.B},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "cpu_model": cpu_model(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as tdist

    from paper_2406_13191_b200 import dual

    rank, world, local = dist_env()
    if world > 1:
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    form = {"F2": dual.FORM_F2, "F1": dual.FORM_F1, "KVL": dual.FORM_KVL, "PTDF": dual.FORM_PTDF}[args.form]
    config, quad, B_total = WORKLOADS[args.workload]
    if args.batch is not None and B_total > 1:
        B_total = int(args.batch)
    if form == dual.FORM_PTDF and args.workload == "config4":
        raise SystemExit("--form PTDF takes load-only batches: use --workload config4b (config 4 has outages)")
    if B_total > 1 and args.scaling == "weak":
        # weak scaling (independent instances, no data-path collective): every
        # rank iterates its own configs[4]-sized batch; rank r takes instances
        # [r B, (r+1) B) of the seeded sweep (instance j's data depend only on j)
        lo, hi = rank * B_total, (rank + 1) * B_total
        B_total = B_total * world
    else:
        lo, hi = shard(B_total, rank, world) if B_total > 1 else (0, 1)
    net, batch = make_inputs(args.workload, lo, hi, total=B_total)
    B = batch.B
    path = dual.PATH_BATCHED if B_total > 1 else dual.PATH_CLUSTER
    if form == dual.FORM_PTDF:
        path = dual.PATH_DENSE
    path = {"auto": path, "batched": dual.PATH_BATCHED, "single": dual.PATH_SINGLE,
            "cluster": dual.PATH_CLUSTER, "dense": dual.PATH_DENSE}[args.path]

    # config 4 takes branches out among the non-tree ones only: declaring that
    # lets the library skip the outage test on the (never switched) tree
    sw = None
    if config == 4 and form != dual.FORM_PTDF:
        sw = np.zeros(net.n_branch, np.uint8)
        sw[net.n_tree:] = 1
    ospec, alpha0 = opt_spec(args)
    tv, tc = (int(x) for x in args.tile.split(",")) if args.tile else (0, 0)
    h = dual.DcopfDual(net, form=form, device=local, path=path, switchable=sw, lane_instances=tv, tile_parts=tc)
    if args.opt != "plain":
        h.set_optimizer(ospec["variant"], ospec.get("rho", 0.0), ospec.get("beta1", 0.0), ospec.get("beta2", 0.0),
                        ospec.get("eps", 0.0))
    stream = torch.cuda.current_stream(dev)
    load_dev = torch.from_numpy(np.ascontiguousarray(batch.load.T)).to(dev)
    outs_dev = None if batch.outages is None else torch.from_numpy(batch.outages).to(dev)
    h.set_instance_batch(load_dev, outs_dev, stream=stream)
    info = h.info()
    K, W = args.steps, args.warmup
    alpha = inst.alpha_schedule(max(K, W, 1), alpha0, args.decay)

    def barrier():
        if world > 1:
            tdist.barrier()

    # ---- warm-up (untimed) --------------------------------------------------
    h.iterate(W, alpha, stream=stream)
    torch.cuda.synchronize()

    # ---- timed region: device events on the launching stream ----------------
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h.iterate(K, alpha, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms_max = float(t.item())

    # ---- per-instance results gathered once (NCCL, off the hot loop) ---------
    bound = torch.empty(B, dtype=torch.float64, device=dev)
    best = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    h.get_bound(bound, best, status, stream=stream)
    gather_ms = None
    if world > 1 and B_total > 1:
        torch.cuda.synchronize()
        g0 = time.perf_counter()
        gathered = gather_instance_results([bound, best, status], B_total,  # NCCL, once, off the hot loop
                                           sizes=[hi - lo] * world if args.scaling == "weak" else None)
        torch.cuda.synchronize()
        gather_ms = 1e3 * (time.perf_counter() - g0)
        assert gathered.shape == (3, B_total)

    # ---- time to gap: the workload's full K once, with the
    # oracle's final best (tests/golden/targets.json, tools/make_targets.py) as
    # reference on the sampled instances; the hit iteration is recorded on device
    ttg = None
    if not args.no_gap:
        ttg = time_to_gap(args, h, net, batch, lo, hi, load_dev, outs_dev, stream, world, dev)

    # ---- one instance's time to a TRUE 1e-3 gap (exact optimum) --------------
    ttg_single = None
    if not args.no_gap and B_total == 1 and world == 1:
        ttg_single = single_true_gap(args, h, batch, load_dev, stream)

    # ---- the batched workload's time to a TRUE 1e-3 gap (best route) ----------
    ttg_batched = None
    if (not args.no_gap and world == 1 and args.workload == "config4" and args.form == "F2"
            and args.opt == "plain" and args.batch is None):
        ttg_batched = batched_true_gap(dev, stream)

    # ---- end-to-end through the public API with host buffers -----------------
    e2e = None
    if not args.no_e2e:
        load_host = torch.from_numpy(np.ascontiguousarray(batch.load.T)).pin_memory()
        outs_host = None if batch.outages is None else torch.from_numpy(batch.outages).pin_memory()
        bound_h = torch.empty(B, dtype=torch.float64).pin_memory()
        best_h = torch.empty(B, dtype=torch.float64).pin_memory()
        status_h = torch.empty(B, dtype=torch.int32).pin_memory()
        h2d = load_host.numel() * 8 + (0 if outs_host is None else outs_host.numel() * 4)
        d2h = B * (8 + 8 + 4)
        samples = []
        for _ in range(3):  # the median of three calls (one call is exposed to host-side noise)
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            h.set_instance_batch(load_host, outs_host, stream=stream)
            h.iterate(K, alpha, stream=stream)
            h.get_bound(bound_h, best_h, status_h, stream=stream)
            torch.cuda.synchronize()
            barrier()
            samples.append(time.perf_counter() - t0)
        e2e_s = sorted(samples)[1]
        te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        if world > 1:
            tdist.all_reduce(te, op=tdist.ReduceOp.MAX)
        # one user call sequence solves the batch for K steps: the loads go up once
        # and the bounds come back once per call, i.e. per K steps
        e2e = {"value": B_total * K / float(te.item()), "unit": UNIT, "h2d_bytes_per_step": h2d / max(K, 1),
               "d2h_bytes_per_step": d2h / max(K, 1), "h2d_bytes_per_call": int(h2d),
               "d2h_bytes_per_call": int(d2h), "steps_per_call": K,
               "timed": "set_instance_batch(host pinned) + iterate(K) + get_bound(host), wall clock, max over ranks, "
                        "median of 3 calls", "call_seconds": samples}

    dense = form == dual.FORM_PTDF
    if rank == 0 and dense and B > 4:
        peak_t = fp64_peak_tflops(dev)
    if rank == 0:
        peak, peak_src = peaks()
        inst_it = B_total * K
        value = inst_it / (ms_max / 1e3)
        # algorithmic HBM bytes of the timed launch: K iterations (read + write
        # the multipliers, read the loads) + the final evaluation (reads only)
        n_bm = (info.alg_bytes_per_inst_iter // 8 - 3 * net.n_bus) // 2  # branch-block multipliers per instance
        eval_read = 8 * (2 * net.n_bus + n_bm)
        per_gpu_bytes = B * (info.alg_bytes_per_inst_iter * K + (eval_read if path == dual.PATH_BATCHED else 0))
        if args.opt != "plain":  # the optimiser state rows (1 or 2 per multiplier) are read and written too
            nstate = 2 if args.opt == "adam" else 1
            n_bm = (info.alg_bytes_per_inst_iter // 8 - 3 * net.n_bus) // 2
            per_gpu_bytes += B * K * nstate * 2 * 8 * (net.n_bus + n_bm)
        achieved = per_gpu_bytes / (ms / 1e3) / 1e9  # GB/s on this rank's kernel launches
        traffic = None  # DRAM bytes per launch, from the committed ncu capture (scaled to this launch)
        try:
            prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
            ent = prof.get(f"{args.workload}/{args.form}")
            if ent and ent.get("dram_over_alg"):
                traffic = ent["dram_over_alg"] * per_gpu_bytes
        except Exception:
            pass
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "alg_bytes_per_inst_iter": info.alg_bytes_per_inst_iter, "peak_source": peak_src}
        if dense and B <= 4:  # skinny batch: matrix-vector passes over H_g (HBM-bound)
            single = B == 1 and info.smem_bytes > 0  # the single-read step: H_g read once per step
            per_step = (8.0 if single else 16.0) * net.n_branch * net.n_gen \
                + 8.0 * B * (7 * net.n_branch + 2 * net.n_gen)
            ach = per_step * K / (ms / 1e3) / 1e9
            roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                    "traffic": None, "alg_bytes_per_step": per_step, "peak_source": peak_src,
                    "kernel": ("the whole step (single-read line pass over H_g with the mu step and the H_g^T nu "
                               "accumulation, generator pass, fused finisher)" if single else
                               "the whole step (2 matrix-vector kernels reading H_g, epilogues, fused finisher)")}
        elif dense:  # two GEMMs per step, 2 n_l n_g flops each per instance (the final evaluation not counted)
            flops = 4.0 * net.n_branch * net.n_gen * B * K
            ach_t = flops / (ms / 1e3) / 1e12
            traffic_t = None  # DRAM bytes of the timed launches, from the committed ncu launch list
            try:
                pk = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))["config4b/PTDF"]["per_kernel"]
                if args.workload == "config4b" and B == inst.CONFIG4_BATCH:
                    # per step: every kernel once per column group (two groups on two streams)
                    traffic_t = K * 2 * sum(v["dram_read"] + v["dram_write"] for v in pk.values())
            except Exception:
                pass
            roof = {"bound": "tensor", "achieved": ach_t, "peak": peak_t, "unit": "TFLOP/s", "frac": ach_t / peak_t,
                    "traffic": traffic_t, "traffic_note": "DRAM bytes (ncu) of K steps: GEMM1 + GEMM2 + finisher",
                    "alg_flops_per_inst_iter": 4 * net.n_branch * net.n_gen,
                    "peak_source": "measured live: cuBLAS DGEMM 8192^3 via torch.matmul, best of 5 (fp64)",
                    "kernel": "the whole step (2 fused DMMA GEMMs + the per-instance finisher)"}
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cores = os.cpu_count() or 1
            if dense:
                rate, sample = ptdf_oracle_rate(net, batch, cores, opt=ospec)
            else:
                rate, sample = cpu_oracle_rate(net, batch, form, cores, opt=ospec)
            cpu = {"value": rate, "unit": UNIT, "cores": cores, "cpu_model": cpu_model(), "kind": "oracle",
                   "sample": sample}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms_max / K, "higher_is_better": True,
            "scaling": (args.scaling if B_total > 1 else "replicas"),
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, BASELINE.json recipe)",
            "config": {"workload": args.workload, "form": args.form, "cost": "QP" if quad else "LP",
                       "step": {"variant": args.opt, "alpha": alpha0, "decay": args.decay, **OPTS[args.opt][1]},
                       "n_bus": net.n_bus, "n_branch": net.n_branch, "n_gen": net.n_gen,
                       "B_total": B_total, "B_per_gpu": B,
                       "path": {1: "batched-sweep", 2: "single", 3: "cluster", 4: "dense-gemm"}[path],
                       "cluster_size": info.cluster_size,
                       "tile": {"lane_instances": info.lane_instances, "parts": info.tile_parts,
                                "halo_items": info.halo_items, "steps_per_sweep": info.steps_per_sweep},
                       "kernel": {"grid": info.grid, "threads": info.threads_per_block, "smem": info.smem_bytes,
                                  "chunk": info.chunk, "tile_width": info.tile_width,
                                  "copies_per_sweep": info.copies_per_sweep, "ring_life": info.ring_life,
                                  "smem_slots_lambda": info.ring_bus, "smem_slots_branch": info.ring_branch,
                                  "order_bandwidth": info.bandwidth},
                       "parallelism": f"instance-shard x{world}",
                       "l2": ("inputs larger than L2: state %.2f GB per GPU" %
                              ((info.B_padded * (2 * net.n_bus + 2 * net.n_branch * (1 if form == 0 else 2)
                                                 + net.n_bus) * 8) / 1e9))
                       if B_total > 1 and not dense else ("H_g %.2f GB read %s per step" %
                                                            (8 * net.n_branch * net.n_gen / 1e9,
                                                             "once" if (B == 1 and info.smem_bytes > 0) else "twice")
                                                            if dense else "state on chip (single instance)"),
                       "timed_launches": (f"{(2 if B <= 4 else 3) * (K + 1)} launches: {2 if B <= 4 else 3} per step "
                                          f"({K} steps) + the final evaluation"
                                          if dense else f"1 persistent launch: {K} iterations + final evaluation")},
            "roofline": roof,
            "cpu_baseline": cpu,
            "time_to_gap": ttg,
            "time_to_true_gap_batched": ttg_batched,
            "time_to_true_gap_single": ttg_single,
            "e2e": e2e,
            "gpu_launches": ((2 if B <= 4 else 3) * (K + 1)) if dense else 1,
            "clocks": clk,
            "gather_ms": gather_ms,
        }
        print(json.dumps(line), flush=True)
    h.close()
    if world > 1:
        tdist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
