"""Run tpo_run on a BASELINE config (default small) REPS times (for ncu of any of its kernels)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_11922_b200 as T
from synth import make_config

g = make_config(os.environ.get("CFG", "small"))
dg = T.to_device_graph(g.n, g.m, g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col, device="cuda:0")
X = torch.from_numpy(g.X).cuda()
runner = T.Runner(dg, g.d, g.k, device="cuda:0")
for _ in range(int(os.environ.get("REPS", 2))):
    lab = runner(X, g.alpha, g.T, g.G, 5, 20)
torch.cuda.synchronize()
print("ok", int(lab.max()))
