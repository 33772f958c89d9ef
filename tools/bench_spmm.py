"""Time tpo_propagate under the SpMM variants (TPO_SPMM_VARIANT = SL*10 + MINB) on BASELINE configs;
results must be bit-identical across variants (same per-element summation order)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_11922_b200 as T
from synth import make_config

cfgs = os.environ.get("CFGS", "small").split(",")
variants = [int(v) for v in os.environ.get("VARIANTS", "14,13,23,22,42,82").split(",")]
for cfg in cfgs:
    g = make_config(cfg)
    dg = T.to_device_graph(g.n, g.m, g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col, device="cuda:0")
    X = torch.from_numpy(g.X).cuda()
    ref = None
    for v in variants:
        os.environ["TPO_SPMM_VARIANT"] = str(v)
        for _ in range(2):
            Z, Zh = T.propagate(dg, X, g.alpha, g.T)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            Z, Zh = T.propagate(dg, X, g.alpha, g.T)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        same = "ref" if ref is None else ("bit-identical" if torch.equal(ref, Z) else "DIFFERENT")
        if ref is None:
            ref = Z.clone()
        ts.sort()
        print(f"{cfg} d={g.d} nnz={g.nnz} T={g.T} variant={v}: median {ts[2]:.3f} ms  min {ts[0]:.3f} ms  ({same})", flush=True)
