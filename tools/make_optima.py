#!/usr/bin/env python3
"""Exact LP optima of a stratified sample of config 4b (BASELINE.json configs[4],
variant 4b: one load factor per instance, no outages -- feasible by
construction, reading A-15), for the TRUE time-to-gap measurement
of the batched routes (bench.py time_to_gap(ii)).

Sample: every 16th instance of the 8192 (512 instances, ids 0, 16, ..., 8176):
evenly spread over the seeded sweep.  Each optimum is the exact minimum of
PAPER.md:94-101 (Eq. 1) in sparse B-theta form, solved by scipy HiGHS
(instances.primal_lp) with the implied angle box -- valid for every feasible
flow, so it is the optimum of Eq. 1 itself and of every form's primal (F2, KVL,
PTDF).  Nothing here touches the CUDA path.

  python tools/make_optima.py [--stride 16] [--procs 8]
"""
import argparse
import json
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2406_13191_b200 import instances as inst  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "optima_config4b.json")
_net = None


def _solve(j):
    global _net
    if _net is None:
        _net = inst.make_network(4)
    b = inst.config4_batch(_net, [int(j)], variant="4b")
    st, obj = inst.primal_lp(_net, b.load[0])
    return int(j), int(st), float(obj)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stride", type=int, default=16)
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    ids = np.arange(0, inst.CONFIG4_BATCH, a.stride)
    t0 = time.time()
    with Pool(a.procs) as pool:
        res = pool.map(_solve, ids, chunksize=4)
    res.sort()
    assert all(st == 0 for _, st, _ in res), "a 4b instance is not optimal (it is feasible by construction)"
    js = {"workload": "config4b", "instance_ids": [j for j, _, _ in res], "primal_opt": [o for _, _, o in res],
          "stride": a.stride, "solver": "scipy.optimize.linprog(method='highs') on the B-theta LP (instances.primal_lp)",
          "note": "exact LP optimum of PAPER.md Eq. 1 per sampled instance; the true-gap reference"}
    json.dump(js, open(OUT, "w"), indent=0)
    print(f"{len(res)} optima in {time.time() - t0:.0f} s -> {OUT}")


if __name__ == "__main__":
    main()
