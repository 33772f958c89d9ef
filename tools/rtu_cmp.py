import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2405_11922_b200 as T
from synth import make_config
g = make_config(os.environ.get("CFG", "small"))
dg = T.to_device_graph(g.n, g.m, g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col)
X = torch.from_numpy(g.X).cuda()
r = T.Runner(dg, g.d, g.k)
for _ in range(3): lab = r(X, g.alpha, g.T, g.G)
torch.cuda.synchronize()
np.save(os.environ["OUT"], lab.cpu().numpy())
print("timings", r.timings)
