"""Measurement only: how fast the dense-PTDF dual (the paper's formulation)
closes the gap on a single instance with each step variant, on the GPU.
Prints best/opt at checkpoints; opt = HiGHS LP optimum of Eq. 1 (no angle box)."""
import dataclasses
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2406_13191_b200 import dual, instances as inst

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
quad = len(sys.argv) > 2 and sys.argv[2] == "qp"
net = inst.make_network(cfg, quadratic=quad)
th = np.full(net.n_bus, 1e6)
th[net.ref_bus] = 0.0
t0 = time.time()
if quad:
    opt = inst.primal_qp(dataclasses.replace(net, theta_max=th), net.base_load)[2]
else:
    opt = inst.primal_lp(dataclasses.replace(net, theta_max=th), net.base_load)[1]
print("opt", opt, "(%.1fs)" % (time.time() - t0), flush=True)
K = int(__import__("os").environ.get("PTDF_K", "5000"))
marks = [m for m in [50, 100, 200, 500, 1000, 2000, 5000, 10000, 20000, 50000] if m <= K]
h = dual.DcopfDual(net, form=dual.FORM_PTDF)
ld = np.ascontiguousarray(net.base_load[:, None])
for name, var, kw, alphas in [("adam", dual.OPT_ADAM, dict(beta1=0.9, beta2=0.999, epsilon=1e-8), [0.01, 0.1, 1.0, 10.0]),
                              ("gdm", dual.OPT_GDM, dict(momentum=0.9), [1e-4, 1e-3, 1e-2]),
                              ("adagrad", dual.OPT_ADAGRAD, dict(epsilon=1e-8), [0.1, 1.0, 10.0, 100.0]),
                              ("plain", dual.OPT_PLAIN, {}, [1e-4, 1e-3, 1e-2])]:
    for a in alphas:
        h.set_optimizer(var, **kw)
        h.set_instance_batch(ld)
        hist = torch.empty((K, 1), dtype=torch.float64, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h.iterate(K, np.full(K, a), hist)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        hh = hist[:, 0].cpu().numpy()
        run = np.maximum.accumulate(np.where(np.isfinite(hh), hh, -np.inf))
        gaps = [(opt - run[m - 1]) / abs(opt) for m in marks]
        first = np.argmax(run >= opt - 1e-3 * abs(opt)) if np.any(run >= opt - 1e-3 * abs(opt)) else -1
        print(f"{name:8s} a={a:<8g} {ms*1e3:7.1f} us/it  gap@" + " ".join(f"{m}:{g:.2e}" for m, g in zip(marks, gaps))
              + f"  first<=1e-3 at k={first}", flush=True)
