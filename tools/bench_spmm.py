"""Time tpo_propagate under the SpMM layouts (TPO_SPMM_L = "Lp,Lq": column-group widths in float4 of
the iterate P and of the V-side block Q; "0,0" = the row-major slice kernel) and the group
kernel's (loads in flight, blocks/SM) configuration (TPO_GSPMM_CFG) on BASELINE configs.  The
group kernels sum in a different (fixed) order than the row-major kernel: results agree to fp32
rounding (relF printed vs the row-major layout)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_11922_b200 as T
from synth import make_config

cfgs = os.environ.get("CFGS", "large").split(",")
layouts = os.environ.get("LAYOUTS", "0,0;auto;8,8;4,4;4,8;8,16;16,16").split(";")
gcfgs = os.environ.get("GCFGS", "0,1").split(",")
# row-major layout: TPO_SPMM_TMA (0 = register gathers, 1 = TMA gather4 ring) x TPO_TG_CFG
tmas = os.environ.get("TMAS", "0").split(",")
tgcfgs = os.environ.get("TGCFGS", "0").split(",")
hots = os.environ.get("HOTS", "0").split(",")        # TPO_SPMM_HOT: MB of hot gathered rows kept evict_last
for cfg in cfgs:
    g = make_config(cfg)
    dg = T.to_device_graph(g.n, g.m, g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col, device="cuda:0")
    X = torch.from_numpy(g.X).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
    ref = None
    combos = [(lay, gc, tm, tg) for lay in layouts for gc in gcfgs for tm in tmas for tg in tgcfgs
              if (lay == "0,0" and gc == gcfgs[0] and (tm == "1" or tg == tgcfgs[0]))
              or (lay != "0,0" and tm == tmas[0] and tg == tgcfgs[0])]
    combos = [(lay, gc, tm, tg, h) for (lay, gc, tm, tg) in combos for h in hots if h == hots[0] or lay == "0,0"]
    for lay, gc, tm, tg, h in combos:
        if True:
            os.environ["TPO_SPMM_HOT"] = h
            os.environ["TPO_SPMM_TMA"] = tm
            os.environ["TPO_TG_CFG"] = tg
            if lay == "auto":
                os.environ.pop("TPO_SPMM_L", None)
            else:
                os.environ["TPO_SPMM_L"] = lay
            os.environ["TPO_GSPMM_CFG"] = gc
            Z, Zh = T.propagate(dg, X, g.alpha, g.T)
            torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                Z, Zh = T.propagate(dg, X, g.alpha, g.T, Z=Z, Zhat=Zh)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            if ref is None:
                ref = Z.clone()
                rel = 0.0
            else:
                rel = float(torch.linalg.norm((Z - ref).double()) / torch.linalg.norm(ref.double()))
            ts.sort()
            print(f"{cfg} d={g.d} nnz={g.nnz} T={g.T} layout={lay} hot={h}: median {ts[2]:.3f} ms  min {ts[0]:.3f} ms "
                  f"per hop {ts[2] / g.T:.3f} ms  relF vs row-major {rel:.2e}", flush=True)
