"""Measurement only: step schedules for the dense-PTDF dual + Adam on one
instance (GPU): gap to the HiGHS optimum of Eq. 1 (no angle box) over k."""
import dataclasses
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2406_13191_b200 import dual, instances as inst

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
qp = len(sys.argv) > 3 and sys.argv[3] == "qp"
net = inst.make_network(cfg, quadratic=qp)
th = np.full(net.n_bus, 1e6)
th[net.ref_bus] = 0.0
if qp:  # Kelley cutting planes: the optimum to ~1e-10 (its upper bound is used)
    opt = inst.primal_qp(dataclasses.replace(net, theta_max=th), net.base_load)[2]
else:
    opt = inst.primal_lp(dataclasses.replace(net, theta_max=th), net.base_load)[1]
print("config", cfg, "opt", opt, flush=True)
k = np.arange(K, dtype=np.float64)
S = {
    "a1": np.full(K, 1.0),
    "a0.5": np.full(K, 0.5),
    "a2/sqrt(k/500)": 2.0 / np.sqrt(1 + k / 500),
    "a1/sqrt(k/1000)": 1.0 / np.sqrt(1 + k / 1000),
    "a3/sqrt(k/200)": 3.0 / np.sqrt(1 + k / 200),
    "a5/(k/200)": 5.0 / (1 + k / 200),
    "a2 step x0.5/2000": 2.0 * 0.5 ** np.floor(k / 2000),
    "a1 step x0.5/3000": 1.0 * 0.5 ** np.floor(k / 3000),
}
marks = [m for m in [100, 200, 500, 1000, 2000, 5000, 10000, 20000, 50000] if m <= K]
h = dual.DcopfDual(net, form=dual.FORM_PTDF)
ld = np.ascontiguousarray(net.base_load[:, None])
for name, a in S.items():
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
    print(f"{name:20s} {dt / K * 1e6:6.1f} us/it  " + " ".join(f"{m}:{g:.1e}" for m, g in zip(marks, gaps))
          + f"  1e-3 at k={first}" + (f" ({first * dt / K * 1e3:.1f} ms)" if first >= 0 else ""), flush=True)
