"""Run tpo_cluster once on small-config-shaped random inputs (for ncu of the skinny products)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2405_11922_b200 as T

n, D, k = int(os.environ.get("N", 50000)), int(os.environ.get("D", 2000)), int(os.environ.get("K", 10))
g = torch.Generator(device="cuda").manual_seed(0)
Rp = (torch.rand(n, D, device="cuda", generator=g) - 0.3) * 0.05
dinv = torch.rand(n, device="cuda", generator=g) + 0.5
Gm = torch.rand(n, k, device="cuda", generator=g) / np.sqrt(n)
Ps = torch.rand(D, k, device="cuda", generator=g) / np.sqrt(D)
sig = np.linspace(1.0, 0.1, k)
for _ in range(2):
    lab, it = T.cluster(Rp, dinv, Gm, sig, Ps, 5, 20)
torch.cuda.synchronize()
print("ok", it)
