"""Debug: where the library's H_a differs from the oracle's (measurement/debug only)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import oracle
from oracle import ptdf as P
from paper_2406_13191_b200 import dual, instances as inst
net = inst.make_network(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
h = dual.DcopfDual(net, form=dual.FORM_PTDF)
H = h.get_ptdf()
Ho = P.ptdf(net)
D = np.abs(H - Ho)
bad = np.argwhere(D > 1e-9)
print("n bad", len(bad), "rows", len(np.unique(bad[:, 0])), "cols", len(np.unique(bad[:, 1])))
rows = np.unique(bad[:, 0])
print("bad rows tree?", [(int(r), int(r < net.n_tree)) for r in rows[:20]])
cols = np.unique(bad[:, 1])
print("bad cols", cols[:40], cols.max() if len(cols) else None)
E = P.incidence(net)
want = np.eye(net.n_bus); want[net.ref_bus, :] -= 1
print("KCL err lib", np.abs(E.T @ H - want).max(), "orc", np.abs(E.T @ Ho - want).max())
_, cyc = oracle.cycles(net)
kv = max(np.abs((sg[:, None] * H[br] / net.br_b[br][:, None]).sum(0)).max() for br, sg in cyc)
print("KVL err lib", kv)
