# measurement only: skinny-mode time per step vs batch size (config 3)
for B in 1 2 4 8 16 17; do
python - <<PY
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2406_13191_b200 import dual, instances as inst
net = inst.make_network(3)
B = $B
loads = net.base_load[:, None] * np.random.default_rng(1).uniform(0.85, 1.15, (1, B))
h = dual.DcopfDual(net, form=dual.FORM_PTDF)
h.set_optimizer(dual.OPT_ADAM, beta1=0.9, beta2=0.999, epsilon=1e-8)
h.set_instance_batch(torch.from_numpy(np.ascontiguousarray(loads)).cuda())
K = 200
h.iterate(10, np.full(10, 1.0)); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); h.iterate(K, np.full(K, 1.0)); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
print(f"B={B} {ms*1e3:.1f} us/step {B / ms * 1e3:.3g} inst-it/s")
PY
done
