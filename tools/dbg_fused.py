import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2406_13191_b200 import dual
from paper_2406_13191_b200 import instances as inst
def run(net, fused, K, opt=False, alpha=1e-3, split=None):
    os.environ["DCOPF_PTDF_FUSED"] = "1" if fused else "0"
    h = dual.DcopfDual(net, form=dual.FORM_PTDF, path=dual.PATH_DENSE)
    if opt: h.set_optimizer(dual.OPT_ADAM, 0.0, 0.9, 0.999, 1e-8)
    h.set_instance_batch(np.ascontiguousarray(net.base_load[:, None]))
    a = inst.alpha_schedule(K, alpha)
    hist = np.empty((K, 1)) if K else None
    if split:
        h.iterate(split, a[:split]); h.iterate(K - split, a[split:])
    else:
        h.iterate(K, a, hist)
    bound, best, status, lam, br = h.results_numpy()
    h.close()
    return bound[0], lam[0, 0], br[:, 0], hist
for cfg in [1, 3]:
    net = inst.make_network(cfg)
    for K in [0, 1, 2, 3, 10, 50]:
        for opt in [False, True]:
            f = run(net, True, K, opt); t = run(net, False, K, opt)
            print(cfg, K, opt, f[0], t[0], f[1], t[1], np.abs(f[2]-t[2]).max() if K else 0, flush=True)
