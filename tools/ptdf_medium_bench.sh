# measurement only: PTDF GEMM mode at medium batch sizes, split-K on / off
for B in 128 512 1024; do
  for sk in 1 0; do
    DCOPF_PTDF_SPLITK=$sk python - <<PY
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
from paper_2406_13191_b200 import dual, instances as inst
net = inst.make_network(3)
B = $B
loads = net.base_load[:, None] * np.random.default_rng(1).uniform(0.85, 1.15, (1, B))
h = dual.DcopfDual(net, form=dual.FORM_PTDF)
h.set_instance_batch(torch.from_numpy(np.ascontiguousarray(loads)).cuda())
K = 20
h.iterate(3, np.full(3, 1e-3)); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); h.iterate(K, np.full(K, 1e-3)); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
print(f"B={B} splitk=$sk {ms:.3f} ms/it {B / ms * 1e3:.3g} inst-it/s")
PY
  done
done
