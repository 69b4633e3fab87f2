import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from paper_2406_13191_b200 import dual, instances as inst
from gpu_helpers import run_gpu, non_tree_switchable
K = int(sys.argv[1]); B = int(sys.argv[2]); cfg = sys.argv[3]
net = inst.tiny_network(23, 37, 30, seed=5) if cfg == "tiny" else inst.make_network(int(cfg))
sw = non_tree_switchable(net)
loads = np.tile(net.base_load[None, :], (B, 1))
a = inst.alpha_schedule(max(K, 1), 4e-3)
g = run_gpu(net, loads, K=K, alpha=a, form=dual.FORM_KVL, path=dual.PATH_BATCHED, switchable=sw)
print("ok", K, B, cfg, g["bound"][:3], g["info"].tile_width, g["info"].chunk, g["info"].smem_bytes)
