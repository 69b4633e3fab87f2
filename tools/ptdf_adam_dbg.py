"""Debug (measurement only): which PTDF multipliers differ GPU vs oracle under Adam."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import ptdf as P
from paper_2406_13191_b200 import dual, instances as inst
from gpu_helpers import run_gpu
net = inst.make_network(1)
Ha = P.ptdf(net)
Hg = Ha[:, net.gen_bus]
K = int(sys.argv[1]) if len(sys.argv) > 1 else 300
a = inst.alpha_schedule(K, 0.1)
loads = net.base_load[None, :] * 1.0
ADAM = dict(variant=P.OPT_ADAM, beta1=0.9, beta2=0.999, eps=1e-8)
g = run_gpu(net, loads, K=K, alpha=a, form=dual.FORM_PTDF, path=dual.PATH_DENSE, history=True, opt=ADAM)
o = P.solve(net, loads, K, a, Ha=Ha, history=True, opt=ADAM)
print("bound", g["bound"], o.bound, "hist maxrel", np.max(np.abs(g["hist"] - o.hist[:, :K]) / np.abs(o.hist[:, :K]).clip(1)))
d = np.abs(g["br"][0] - o.mu[0])
nl = net.n_branch
idx = np.argsort(-d)[:10]
r = Ha @ loads[0]
for i in idx:
    l = i % nl
    print(i, "mu+" if i < nl else "mu-", "diff %.3g" % d[i], "gpu %.6g orc %.6g" % (g["br"][0][i], o.mu[0][i]), "F", net.br_fmax[l], "Hg0", np.max(np.abs(Hg[l])) < 1e-12, "r %.3g" % r[l])
print("lam", g["lam"][0], o.lam[0])
for k in (10, 50, 100, 200, K - 1):
    kk = min(k, K - 1)
    print(k, "hist gpu %.12g orc %.12g" % (g["hist"][0, kk], o.hist[0, kk]))
