"""Debug dump of the tcgen05 Gram kernel on a tiny constant input."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import torch
import paper_2405_11922_b200 as T
from paper_2405_11922_b200._lib import lib
L = lib()
dbg = torch.zeros(256, dtype=torch.float32, device="cuda")
L.tpo__gram_debug.argtypes = [C.c_void_p]
L.tpo__gram_debug(C.c_void_p(dbg.data_ptr()))
n, D = 64, 128
Rp = (torch.arange(n * D, device="cuda", dtype=torch.float32).reshape(n, D) % 7 + 1) / 8
dinv = torch.ones(n, device="cuda")
G = T.gram(Rp, dinv)
torch.cuda.synchronize()
d = dbg.cpu().numpy()
print("smem A_hi row0[0:32]", d[:32])
print("smem A_lo row0[0:32]", d[32:64])
print("smem A_hi +128B", d[64:96])
print("tmem lane0 cols0..31", d[96:128])
print("tmem_base bits", np.frombuffer(d[128:129].tobytes(), np.uint32), "nkb", d[129], "nseg", d[130])
ref = (Rp.double().T @ Rp.double()).cpu().numpy()
print("G[0,:8]", G[0, :8].cpu().numpy(), "ref", ref[0, :8])
print("maxerr", np.abs(G.cpu().numpy() - ref).max())
