"""Run the device Haar rotation (d = 1000 by default) twice (for ncu of its kernels)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2405_11922_b200 as T

d = int(os.environ.get("D", 1000))
G = np.random.default_rng(0).standard_normal((d, d))
for _ in range(2):
    Q = T.haar_q_dev(G)
torch.cuda.synchronize()
print("ok", float(Q.norm()))
