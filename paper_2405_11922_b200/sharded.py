"""Multi-GPU MSA propagation: U rows sharded across ranks.

One process per GPU.  Rank p owns the contiguous U slice [u0, u1) of the ABG: CSR(B_p) (its rows
of B, global V ids) and CSR(B_p^T) (m x n_p, local U ids).  Per hop (Eq. update-Z, PAPER.md:454,
bracketed L (L^T Z) as PAPER.md:456):

    Qpart  = B_p^T P_p                       (libtpo: tpo_shard_vside; m x d partial)
    Qslice = reduce-scatter(sum) over V      (NCCL via torch.distributed)
    Qslice *= s_v^2                          (libtpo: tpo_shard_vscale)
    Q      = all-gather(Qslice)              (NCCL)
    P_p    = s_u (c X_p + alpha s_u B_p Q)   (libtpo: tpo_shard_uside; last hop: Z_p, Zhat_p)

plus one all-reduce of the V-side degree partials.  Summing the shard partials of
B^T (s_u . Z) over ranks is the full product, so the result is tpo_propagate's.

The orchestration takes its local compute (`ops`) and its collectives (`coll`) as objects, so
the exchange algebra is exercised on CPU with gloo in tests/test_sharded.py; GpuShardOps is the
only implementation used on GPUs.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from ._lib import CSR, check, lib


@dataclass
class HostShard:
    """One rank's share of an ABG (host arrays)."""
    rank: int
    world: int
    n: int            # global |U|
    m: int            # global |V|
    u0: int
    u1: int
    Bp_rowptr: np.ndarray
    Bp_col: np.ndarray
    Btp_rowptr: np.ndarray
    Btp_col: np.ndarray
    Bp_val: Optional[np.ndarray] = None
    Btp_val: Optional[np.ndarray] = None

    @property
    def n_p(self) -> int:
        return self.u1 - self.u0

    @property
    def nnz(self) -> int:
        return int(self.Bp_col.shape[0])


def row_bounds(n: int, rank: int, world: int):
    return (n * rank) // world, (n * (rank + 1)) // world


def shard_graph(n, m, B_rowptr, B_col, rank, world, B_val=None) -> HostShard:
    """Cut the contiguous U slice of `rank` out of the global CSR(B) and transpose it locally."""
    u0, u1 = row_bounds(n, rank, world)
    e0, e1 = int(B_rowptr[u0]), int(B_rowptr[u1])
    rp = (np.asarray(B_rowptr[u0:u1 + 1], np.int64) - e0).astype(np.int64)
    col = np.ascontiguousarray(B_col[e0:e1], np.int32)
    val = None if B_val is None else np.ascontiguousarray(B_val[e0:e1], np.float32)
    n_p = u1 - u0
    u_loc = np.repeat(np.arange(n_p, dtype=np.int64), np.diff(rp))
    order = np.lexsort((u_loc, col.astype(np.int64)))
    t_col = u_loc[order].astype(np.int32)
    t_rp = np.zeros(m + 1, np.int64)
    np.cumsum(np.bincount(col, minlength=m), out=t_rp[1:])
    t_val = None if val is None else np.ascontiguousarray(val[order])
    return HostShard(rank, world, n, m, u0, u1, rp, col, t_rp, t_col, val, t_val)


class TorchCollectives:
    """Collectives over a torch.distributed process group (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.backend = dist.get_backend(group)

    def allreduce_sum(self, t: torch.Tensor):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)

    def reduce_scatter_sum(self, out: torch.Tensor, inp: torch.Tensor):
        if self.backend == "nccl":
            self.dist.reduce_scatter_tensor(out, inp, op=self.dist.ReduceOp.SUM, group=self.group)
        else:
            tmp = inp.clone()
            self.dist.all_reduce(tmp, op=self.dist.ReduceOp.SUM, group=self.group)
            rows = out.shape[0]
            out.copy_(tmp[self.rank * rows:(self.rank + 1) * rows])

    def all_gather(self, out: torch.Tensor, inp: torch.Tensor):
        if self.backend == "nccl":
            self.dist.all_gather_into_tensor(out, inp, group=self.group)
        else:
            parts = list(out.chunk(self.world, dim=0))
            self.dist.all_gather(parts, inp.contiguous(), group=self.group)


class GpuShardOps:
    """Local compute of one shard through libtpo's tpo_shard_* entry points (device tensors)."""

    def __init__(self, shard: HostShard, device, d: int):
        self.s = shard
        self.device = torch.device(device)
        self.d = d

        def dev(a, dt):
            return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(self.device, dt)
        self.Bp = (dev(shard.Bp_rowptr, torch.int64), dev(shard.Bp_col, torch.int32), dev(shard.Bp_val, torch.float32))
        self.Btp = (dev(shard.Btp_rowptr, torch.int64), dev(shard.Btp_col, torch.int32),
                    dev(shard.Btp_val, torch.float32))
        L = lib()
        nb = max(L.tpo_shard_ws(shard.n_p, shard.nnz, d), L.tpo_shard_ws(shard.m, shard.nnz, d))
        self.ws = torch.empty(max(int(nb), 256), dtype=torch.uint8, device=self.device)

    def _csr(self, which):
        s = self.s
        if which == "B":
            rp, col, val = self.Bp
            return CSR(s.n_p, s.m, s.nnz, rp.data_ptr(), col.data_ptr(), None if val is None else val.data_ptr())
        rp, col, val = self.Btp
        return CSR(s.m, s.n_p, s.nnz, rp.data_ptr(), col.data_ptr(), None if val is None else val.data_ptr())

    @staticmethod
    def _p(t):
        return None if t is None else C.c_void_p(t.data_ptr())

    def _st(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def new(self, rows, cols=None, dtype=torch.float32, zero=False):
        shape = (rows,) if cols is None else (rows, cols)
        f = torch.zeros if zero else torch.empty
        return f(shape, dtype=dtype, device=self.device)

    def propagate_local(self, Xp, alpha, T):
        """tpo_propagate on the shard's own rows (used for T = 0, where no exchange is needed)."""
        from .tpo import DeviceGraph, propagate
        g = DeviceGraph(self.s.n_p, self.s.m, self.s.nnz, self.Bp[0], self.Bp[1], self.Btp[0], self.Btp[1],
                        self.Bp[2], self.Btp[2])
        return propagate(g, Xp, alpha, T)

    def degrees(self):
        du = self.new(self.s.n_p, dtype=torch.float64)
        dv = self.new(self.s.m, dtype=torch.float64)
        B, Bt = self._csr("B"), self._csr("Bt")
        check(lib().tpo_shard_degrees(C.byref(B), C.byref(Bt), self._p(du), self._p(dv), self._st()))
        return du, dv

    def start(self, du, dv, Xp, alpha):
        s_u = self.new(self.s.n_p)
        s_v = self.new(self.s.m)
        P = self.new(self.s.n_p, self.d)
        check(lib().tpo_shard_start(self._p(du), self._p(dv), self.s.n_p, self.s.m, self._p(Xp), self.d, float(alpha),
                                    self._p(s_u), self._p(s_v), self._p(P), self._st()))
        return s_u, s_v, P

    def vside(self, P, Qpart):
        Bt = self._csr("Bt")
        check(lib().tpo_shard_vside(C.byref(Bt), self._p(P), self.d, self._p(Qpart), self._p(self.ws), self.ws.numel(),
                                    self._st()))

    def vscale(self, Q, s_v):
        check(lib().tpo_shard_vscale(self._p(Q), self._p(s_v), Q.shape[0], self.d, self._st()))

    def uside(self, Q, Xp, alpha, s_u, last, Zp, Zhat):
        B = self._csr("B")
        check(lib().tpo_shard_uside(C.byref(B), self._p(Q), self._p(Xp), self.d, float(alpha), self._p(s_u),
                                    int(bool(last)), self._p(Zp), self._p(Zhat), self._p(self.ws), self.ws.numel(),
                                    self._st()))


def propagate_sharded(ops, coll, Xp: torch.Tensor, alpha: float, T: int, want_zhat: bool = True):
    """Sharded a1-a3 on this rank: returns (Z_p, Zhat_p) for the rank's U rows."""
    s = ops.s
    n_p, m, d = s.n_p, s.m, Xp.shape[1]
    world = coll.world
    if T == 0:                                               # Z = (1 - alpha) X: rows are independent
        return ops.propagate_local(Xp, alpha, 0)
    du, dv = ops.degrees()
    coll.allreduce_sum(dv)                                   # global D_V
    s_u, s_v, P = ops.start(du, dv, Xp, alpha)
    mp = -(-m // world)                                      # V rows per rank after padding
    m_pad = mp * world
    s_v_pad = ops.new(m_pad, zero=True)
    s_v_pad[:m] = s_v
    Qpart = ops.new(m_pad, d, zero=True)                     # rows >= m stay zero
    Qslice = ops.new(mp, d)
    Q = ops.new(m_pad, d)
    Z = P                                                    # the iterate lives in P's buffer
    Zhat = ops.new(n_p, d) if want_zhat else None
    for t in range(T):
        ops.vside(P, Qpart[:m] if m_pad != m else Qpart)
        coll.reduce_scatter_sum(Qslice, Qpart)
        ops.vscale(Qslice, s_v_pad[coll.rank * mp:(coll.rank + 1) * mp])
        coll.all_gather(Q, Qslice)
        last = t == T - 1
        ops.uside(Q, Xp, alpha, s_u, last, Z, Zhat if last else None)
    return Z, Zhat
