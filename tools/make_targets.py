#!/usr/bin/env python3
"""Reference bounds for the time-to-gap measurement.

For each benched workload and form, runs the ORACLE (oracle/, fp64 CPU) for
the workload's K (BASELINE.json configs: 20000 / 20000 / 50000 / 5000) with
the fixed step alpha = 1e-3 (reading A-9) and stores its final running best
bound per sampled instance in tests/golden/targets.json.  bench.py reads the
file and asks the library for the first iteration at which the GPU's running
best reaches (1 - 1e-3) of it (on the sign-aware side).  Config 4 uses the
deterministic sample of every 128th instance (64 instances), as SURVEY.md
§8(d) prescribes for the oracle at that size.

Form PTDF (oracle/ptdf.py): config 4b only (load-only batch),
16 sampled instances (every 512th); the true gap is taken against the LP
optimum of Eq. 1 itself, i.e. without an angle box (HiGHS on B-theta with
Theta = inf, which never touches H).

Calls only oracle/ and the seeded input generator; nothing here comes from
the CUDA path.

  python tools/make_targets.py [--only config4/F2 ...] [--threads N]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2406_13191_b200 import instances as inst  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "targets.json")
WORKLOADS = {"config1": (1, False), "config2": (2, True), "config3": (3, False), "config3q": (3, True),
             "config4": (4, False), "config4b": (4, False)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--opt", default="plain", help="ascent-step variant (bench.py OPTS)")
    ap.add_argument("--alpha", type=float, default=None)
    ap.add_argument("--workloads", nargs="*", default=None)
    ap.add_argument("--forms", nargs="*", default=["F2", "F1"])
    ap.add_argument("--decay", default=None, help="step decay (instances.alpha_schedule)")
    ap.add_argument("--K", type=int, default=None, help="override the workload's K")
    a = ap.parse_args()
    js = json.load(open(OUT)) if os.path.exists(OUT) else {}
    import bench
    v, hp, a0 = bench.OPTS[a.opt]
    alpha = a.alpha if a.alpha is not None else a0
    opt = dict(variant=v, **hp)
    for wl, (config, quad) in WORKLOADS.items():
        if a.workloads and wl not in a.workloads:
            continue
        for form_name, form in (("F2", oracle.FORM_F2), ("F1", oracle.FORM_F1), ("KVL", oracle.FORM_KVL),
                                ("PTDF", None)):
            if form_name not in a.forms:
                continue
            key = (f"{wl}/{form_name}" + ("" if a.opt == "plain" else f"/{a.opt}/{alpha:g}")
                   + (f"/{a.decay}" if a.decay else ""))
            if a.only and key not in a.only:
                continue
            if form_name == "PTDF" and wl not in ("config4b", "config1", "config3"):
                continue
            net = inst.make_network(config, quadratic=quad)
            K = a.K or inst.ITERS[config]
            if form_name == "PTDF":
                import dataclasses
                from oracle import ptdf as P
                if config == 4:
                    ids = np.arange(0, inst.CONFIG4_BATCH, 512)
                    batch = inst.config4_batch(net, ids, variant="4b")
                else:
                    ids = np.zeros(1, dtype=np.int64)
                    batch = inst.single_batch(net)
                t0 = time.time()
                res = P.solve(net, batch.load, K, inst.alpha_schedule(K, alpha, a.decay), opt=opt)
                th = np.full(net.n_bus, 1e6)
                th[net.ref_bus] = 0.0
                nob = dataclasses.replace(net, theta_max=th)
                primal = [inst.primal_lp(nob, batch.load[r])[1] for r in range(len(ids))]
                js[key] = {"K": K, "alpha": alpha, "decay": a.decay, "opt": {"name": a.opt, **opt},
                           "primal_opt": primal if config == 4 else primal[0],
                           "primal_note": "LP optimum of Eq. 1 (no angle box)",
                           "instance_ids": ids.tolist(), "best": res.best.tolist(), "bound": res.bound.tolist(),
                           "status": res.status.tolist(), "source": "oracle/ptdf.py via tools/make_targets.py"}
                print(key, f"{time.time() - t0:.1f}s", "best[:4] =", res.best[:4], flush=True)
                json.dump(js, open(OUT, "w"), indent=0)
                continue
            if config == 4:
                ids = np.arange(0, inst.CONFIG4_BATCH, 128)
                batch = inst.config4_batch(net, ids, variant="4b" if wl == "config4b" else "4")
            else:
                ids = np.zeros(1, dtype=np.int64)
                batch = inst.single_batch(net)
            t0 = time.time()
            sw = None
            if config == 4:  # only non-tree branches are ever taken out (bench.py passes the same mask)
                sw = np.zeros(net.n_branch, np.uint8)
                sw[net.n_tree:] = 1
            res = oracle.solve(net, batch.load, outages=batch.outages, K=K, alpha=inst.alpha_schedule(K, alpha, a.decay),
                               form=form, threads=a.threads, opt=opt, switchable=sw)
            primal = None
            if config != 4:  # the exact optimum (HiGHS; Kelley cutting planes for QP): true gap, (ii)
                primal = (inst.primal_qp(net, net.base_load) if quad else inst.primal_lp(net, net.base_load))[1]
            elif wl == "config4b":  # feasible instances: their LP optima (sampled)
                primal = [inst.primal_lp(net, batch.load[r])[1] for r in range(len(ids))]
            js[key] = {"K": K, "alpha": alpha, "opt": {"name": a.opt, **opt}, "primal_opt": primal,
                       "instance_ids": ids.tolist(), "best": res.best.tolist(),
                       "bound": res.bound.tolist(), "status": res.status.tolist(),
                       "source": "oracle/dcopf_oracle.c via tools/make_targets.py"}
            print(key, f"{time.time() - t0:.1f}s", "best[:4] =", res.best[:4], flush=True)
            json.dump(js, open(OUT, "w"), indent=0)


if __name__ == "__main__":
    main()
