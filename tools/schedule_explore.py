"""Measurement only: gap to the HiGHS optimum over k for a form / step variant /
schedule on one instance (GPU).  usage: schedule_explore.py CONFIG FORM K"""
import dataclasses
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2406_13191_b200 import dual, instances as inst

cfg, form, K = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
net = inst.make_network(cfg)
th = np.full(net.n_bus, 1e6)
th[net.ref_bus] = 0.0
nb = dataclasses.replace(net, theta_max=th) if form in ("KVL", "PTDF") else net
opt = inst.primal_lp(nb, net.base_load)[1]
print("config", cfg, form, "opt", opt, flush=True)
fid = {"F2": dual.FORM_F2, "F1": dual.FORM_F1, "KVL": dual.FORM_KVL, "PTDF": dual.FORM_PTDF}[form]
specs = [(0.1, None), (0.3, None), (1.0, "inv:200"), (0.5, "inv:500"), (2.0, "inv:200"), (0.3, "step:0.5:5000"),
         (1.0, "step:0.5:3000"), (5.0, "inv:200")]
marks = [m for m in [100, 500, 1000, 2000, 5000, 10000, 20000, 50000] if m <= K]
h = dual.DcopfDual(net, form=fid)
ld = np.ascontiguousarray(net.base_load[:, None])
for a0, dec in specs:
    a = inst.alpha_schedule(K, a0, dec)
    h.set_optimizer(dual.OPT_ADAM, beta1=0.9, beta2=0.999, epsilon=1e-8)
    h.set_instance_batch(ld)
    hist = torch.empty((K, 1), dtype=torch.float64, device="cuda")
    t0 = time.time()
    h.iterate(K, a, hist)
    torch.cuda.synchronize()
    dt = time.time() - t0
    hh = hist[:, 0].cpu().numpy()
    run = np.maximum.accumulate(np.where(np.isfinite(hh), hh, -np.inf))
    gaps = [(opt - run[m - 1]) / abs(opt) for m in marks]
    hit = np.flatnonzero(run >= opt - 1e-3 * abs(opt))
    first = int(hit[0]) if len(hit) else -1
    print(f"a={a0:<5g} {str(dec):15s} {dt / K * 1e6:6.1f} us/it " + " ".join(f"{m}:{g:.1e}" for m, g in zip(marks, gaps))
          + f"  1e-3 at k={first}" + (f" ({first * dt / K * 1e3:.1f} ms)" if first >= 0 else ""), flush=True)
