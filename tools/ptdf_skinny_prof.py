"""Measurement only: a few PTDF iterations on one config-3 instance (skinny mode), for ncu."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2406_13191_b200 import dual, instances as inst
net = inst.make_network(3)
h = dual.DcopfDual(net, form=dual.FORM_PTDF)
h.set_optimizer(dual.OPT_ADAM, beta1=0.9, beta2=0.999, epsilon=1e-8)
h.set_instance_batch(np.ascontiguousarray(net.base_load[:, None]))
K = int(sys.argv[1]) if len(sys.argv) > 1 else 10
h.iterate(K, np.full(K, 1.0))
b = np.empty(1)
h.get_bound(b)
print("bound", b)
