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

exchange="touched" replaces the reduce-scatter / all-gather of the whole m x d
block by two all-to-all exchanges of only the V rows a rank's U slice touches (the non-empty rows
of B_p^T): partial rows go to their V owner, which adds the ranks' blocks in rank order (fixed
order: deterministic); the owners send back exactly those rows of Q.  On the large config each
of 8 ranks touches ~35 % of V, so the volume drops ~3x.

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

    def all_to_all(self, out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits):
        """Rows of inp split by in_splits go to ranks 0..world-1; out receives out_splits rows from each."""
        self.dist.all_to_all_single(out, inp, [int(x) for x in out_splits], [int(x) for x in in_splits],
                                    group=self.group)

    def all_gather_rows(self, t: torch.Tensor) -> torch.Tensor:
        """(world, *t.shape): every rank's copy of t."""
        out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        if self.backend == "nccl":
            self.dist.all_gather_into_tensor(out.view(-1), t.contiguous().view(-1), group=self.group)
        else:
            self.dist.all_gather([out[r] for r in range(self.world)], t.contiguous(), group=self.group)
        return out


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

    def index(self, ids: np.ndarray) -> torch.Tensor:
        return torch.from_numpy(np.ascontiguousarray(ids, np.int32)).to(self.device)

    def pack(self, src, idx, dst):
        """dst[i] = src[idx[i]] (tpo_rows_gather)."""
        check(lib().tpo_rows_gather(self._p(src), self._p(idx), idx.numel(), self.d, self._p(dst), self._st()))

    def unpack(self, dst, idx, src, accumulate):
        """dst[idx[i]] (+)= src[i] (tpo_rows_scatter)."""
        check(lib().tpo_rows_scatter(self._p(dst), self._p(idx), idx.numel(), self.d, self._p(src), int(bool(accumulate)),
                                     self._st()))

    def uside(self, Q, Xp, alpha, s_u, last, Zp, Zhat):
        B = self._csr("B")
        check(lib().tpo_shard_uside(C.byref(B), self._p(Q), self._p(Xp), self.d, float(alpha), self._p(s_u),
                                    int(bool(last)), self._p(Zp), self._p(Zhat), self._p(self.ws), self.ws.numel(),
                                    self._st()))


class TouchedExchange:
    """Index lists of the touched-row exchange (built once per graph): the V rows this rank's U
    slice touches, grouped by V owner (owner(v) = v // mp), and the rows every other rank sends
    to this owner."""

    def __init__(self, ops, coll, m: int):
        s = ops.s
        world, rank = coll.world, coll.rank
        self.mp = -(-m // world)
        touched = np.flatnonzero(np.diff(s.Btp_rowptr) > 0).astype(np.int64)     # sorted global V ids
        owner = touched // self.mp
        self.send_counts = np.bincount(owner, minlength=world).astype(np.int64)
        sc = torch.from_numpy(self.send_counts.copy())
        rc = torch.empty(world, dtype=torch.int64)
        coll.all_to_all(rc, sc, [1] * world, [1] * world)
        self.recv_counts = rc.numpy().astype(np.int64)
        ids_in = torch.empty(int(self.recv_counts.sum()), dtype=torch.int64)
        coll.all_to_all(ids_in, torch.from_numpy(touched.copy()), self.recv_counts, self.send_counts)
        recv_local = ids_in.numpy() - rank * self.mp                  # rows of this rank's V slice
        self.send_idx = ops.index(touched)                            # rows of Qpart / Q (global V ids)
        off = np.concatenate([[0], np.cumsum(self.recv_counts)])
        self.recv_idx = [ops.index(recv_local[off[q]:off[q + 1]]) for q in range(world)]
        self.recv_idx_all = ops.index(recv_local)
        self.recv_off = off
        self.n_send, self.n_recv = int(self.send_counts.sum()), int(self.recv_counts.sum())

    def reduce(self, ops, coll, Qpart, Qslice, d):
        """Qslice = sum over ranks of their touched partial rows of this owner's V slice."""
        sendbuf = ops.new(self.n_send, d)
        ops.pack(Qpart, self.send_idx, sendbuf)
        recvbuf = ops.new(self.n_recv, d)
        coll.all_to_all(recvbuf, sendbuf, self.recv_counts, self.send_counts)
        Qslice.zero_()
        for q in range(coll.world):                                  # rank order: fixed sums
            a, b = int(self.recv_off[q]), int(self.recv_off[q + 1])
            if b > a:
                ops.unpack(Qslice, self.recv_idx[q], recvbuf[a:b], True)

    def gather(self, ops, coll, Qslice, Q, d):
        """Q[v] for every touched v of this rank, from the owners' scaled slices."""
        sendbuf = ops.new(self.n_recv, d)
        ops.pack(Qslice, self.recv_idx_all, sendbuf)
        recvbuf = ops.new(self.n_send, d)
        coll.all_to_all(recvbuf, sendbuf, self.send_counts, self.recv_counts)
        ops.unpack(Q, self.send_idx, recvbuf, False)


def propagate_sharded(ops, coll, Xp: torch.Tensor, alpha: float, T: int, want_zhat: bool = True,
                      exchange: str = "full"):
    """Sharded a1-a3 on this rank: returns (Z_p, Zhat_p) for the rank's U rows.  exchange = "full"
    (reduce-scatter + all-gather of the m x d block) or "touched" (all-to-all of touched rows only)."""
    s = ops.s
    n_p, m, d = s.n_p, s.m, Xp.shape[1]
    world = coll.world
    if T == 0:                                               # Z = (1 - alpha) X: rows are independent
        return ops.propagate_local(Xp, alpha, 0)
    if exchange == "touched":
        return _propagate_touched(ops, coll, Xp, alpha, T, want_zhat)
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


def _propagate_touched(ops, coll, Xp, alpha, T, want_zhat):
    s = ops.s
    n_p, m, d = s.n_p, s.m, Xp.shape[1]
    du, dv = ops.degrees()
    coll.allreduce_sum(dv)                                   # global D_V
    s_u, s_v, P = ops.start(du, dv, Xp, alpha)
    ex = TouchedExchange(ops, coll, m)
    mp = ex.mp
    v0, v1 = coll.rank * mp, min(m, (coll.rank + 1) * mp)
    s_v_slice = ops.new(mp, zero=True)
    if v1 > v0:
        s_v_slice[:v1 - v0] = s_v[v0:v1]
    Qpart = ops.new(m, d)
    Qslice = ops.new(mp, d)
    Q = ops.new(m, d, zero=True)                              # only the touched rows are read
    Z = P
    Zhat = ops.new(n_p, d) if want_zhat else None
    for t in range(T):
        ops.vside(P, Qpart)
        ex.reduce(ops, coll, Qpart, Qslice, d)
        ops.vscale(Qslice, s_v_slice)
        ex.gather(ops, coll, Qslice, Q, d)
        last = t == T - 1
        ops.uside(Q, Xp, alpha, s_u, last, Z, Zhat if last else None)
    return Z, Zhat


class NcclComm:
    """A libtpo-owned NCCL communicator (tpo_comm_create / tpo_comm_destroy).  `uid` is the 128-byte
    ncclUniqueId rank 0 created with NcclComm.unique_id() and shared with the other ranks."""

    def __init__(self, rank: int, world: int, device, uid: bytes):
        self.rank, self.world = rank, world
        self.device = torch.device(device)
        buf = C.create_string_buffer(bytes(uid), 128)
        h = C.c_void_p()
        check(lib().tpo_comm_create(buf, int(rank), int(world), int(self.device.index or 0), C.byref(h)))
        self.h = h

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().tpo_comm_unique_id(buf))
        return buf.raw

    def close(self):
        if self.h:
            check(lib().tpo_comm_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def propagate_sharded_lib(comm: NcclComm, ops: "GpuShardOps", Xp: torch.Tensor, alpha: float, T: int,
                          want_zhat: bool = True, stream=None):
    """Sharded a1-a3 with the collectives inside libtpo (tpo_propagate_sharded on the library's NCCL
    communicator): returns (Z_p, Zhat_p)."""
    s = ops.s
    d = Xp.shape[1]
    Z = torch.empty_like(Xp)
    Zh = torch.empty_like(Xp) if want_zhat else None
    L = lib()
    ws = torch.empty(max(int(L.tpo_propagate_sharded_ws(s.n_p, s.m, s.nnz, d, comm.world)), 256), dtype=torch.uint8,
                     device=Xp.device)
    B, Bt = ops._csr("B"), ops._csr("Bt")
    st = C.c_void_p((stream or torch.cuda.current_stream(Xp.device)).cuda_stream)
    check(L.tpo_propagate_sharded(comm.h, C.byref(B), C.byref(Bt), ops._p(Xp), d, float(alpha), int(T), ops._p(Z),
                                  ops._p(Zh), ops._p(ws), ws.numel(), st))
    return Z, Zh


class LibRunner:
    """The whole hot path on this rank's U slice with the collectives inside libtpo
    (tpo_run_sharded on a NcclComm).  Workspace and label buffers are kept across calls."""

    def __init__(self, comm: NcclComm, ops: "GpuShardOps", d: int, k: int):
        self.comm, self.ops, self.d, self.k = comm, ops, d, k
        s = ops.s
        L = lib()
        self.ws = torch.empty(max(int(L.tpo_run_sharded_ws(s.n_p, s.m, s.nnz, d, k, comm.world)), 256), dtype=torch.uint8,
                              device=ops.device)
        self.labels = torch.empty(max(s.n_p, 1), dtype=torch.int32, device=ops.device)
        self.timings = np.zeros(4, np.float64)
        self.iters = 0

    def __call__(self, Xp: torch.Tensor, alpha: float, T: int, Gdev: torch.Tensor, Tf: int = 5, Tg: int = 20,
                 stream=None):
        s = self.ops.s
        B, Bt = self.ops._csr("B"), self.ops._csr("Bt")
        it = C.c_int32(0)
        st = C.c_void_p((stream or torch.cuda.current_stream(self.ops.device)).cuda_stream)
        check(lib().tpo_run_sharded(self.comm.h, C.byref(B), C.byref(Bt), self.ops._p(Xp), self.d, float(alpha), int(T),
                                    int(self.k), self.ops._p(Gdev), int(s.u0), int(Tf), int(Tg),
                                    self.ops._p(self.labels), C.byref(it), self.timings.ctypes.data_as(C.c_void_p),
                                    self.ops._p(self.ws), self.ws.numel(), st))
        self.iters = int(it.value)
        return self.labels[: s.n_p]


# ------------------------------------------------------------------------------------------
# a5-a9 on row shards ("an all-reduce of the d x k Gram matrices"): every
# D x D, D x k and k x k quantity is the all-reduced sum of the shards' partials, so each rank
# holds the same replicated factors; the n-row quantities stay on their rank.
# ------------------------------------------------------------------------------------------
class GpuSolverOps:
    """Local compute of the sharded solver through libtpo's tpo_shard_* solver entry points."""

    def __init__(self, n_p: int, d: int, k: int, device):
        self.n_p, self.d, self.k, self.D = n_p, d, k, 2 * d
        self.device = torch.device(device)
        nb = lib().tpo_shard_solver_ws(n_p, d, k)
        nb = max(nb, lib().tpo_gram_ws(max(n_p, 1), self.D))
        self.ws = torch.empty(max(int(nb), 256), dtype=torch.uint8, device=self.device)

    @staticmethod
    def _p(t):
        return None if t is None else C.c_void_p(t.data_ptr())

    def _st(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _z(self, *shape, dtype=torch.float64):
        return torch.zeros(shape, dtype=dtype, device=self.device)

    def _ws(self):
        return self._p(self.ws), self.ws.numel()

    def features(self, Zhat_p, Q):
        Rp = torch.empty(self.n_p, self.D, dtype=torch.float32, device=self.device)
        r = self._z(self.D)
        check(lib().tpo_shard_features(self._p(Zhat_p), self.n_p, self.d, self._p(Q), self._p(Rp), self._p(r),
                                       *self._ws(), self._st()))
        return Rp, r

    def dinv(self, Rp, r):
        dv = torch.empty(self.n_p, dtype=torch.float32, device=self.device)
        check(lib().tpo_shard_dinv(self._p(Rp), self.n_p, self.D, self._p(r), self._p(dv), self._st()))
        return dv

    def gram(self, Rp, dinv):
        G = self._z(self.D, self.D)
        if self.n_p > 0:
            check(lib().tpo_gram(self._p(Rp), self._p(dinv), self.n_p, self.D, self._p(G), *self._ws(), self._st()))
        return G

    def eig(self, G, r):
        Psi64 = self._z(self.D, self.k)
        sig = np.zeros(self.k)
        check(lib().tpo_eig_from_gram(self._p(G), self._p(r), self.D, self.k, self._p(Psi64),
                                      sig.ctypes.data_as(C.c_void_p), *self._ws(), self._st()))
        return Psi64, sig

    def gamma(self, Rp, dinv, Psi64, sigma):
        G64 = self._z(self.n_p, self.k)
        sig = np.ascontiguousarray(sigma, np.float64)
        check(lib().tpo_shard_gamma(self._p(Rp), self._p(dinv), self.n_p, self.D, self.k, self._p(Psi64),
                                    sig.ctypes.data_as(C.c_void_p), self._p(G64), *self._ws(), self._st()))
        return G64

    def atb(self, A, B):
        out = self._z(self.k, self.k)
        check(lib().tpo_shard_atb64(self._p(A), self._p(B), self.n_p, self.k, self._p(out), *self._ws(), self._st()))
        return out

    def apply_chol(self, X, g):
        check(lib().tpo_shard_apply_chol(self._p(X), self.n_p, self.k, self._p(g), *self._ws(), self._st()))

    def colstats(self, G64, row0):
        s, a, v = self._z(self.k), self._z(self.k), self._z(self.k)
        i = torch.zeros(self.k, dtype=torch.int64, device=self.device)
        check(lib().tpo_shard_colstats(self._p(G64), self.n_p, self.k, int(row0), self._p(s), self._p(a), self._p(v),
                                       self._p(i), *self._ws(), self._st()))
        return s, a, v, i

    def gamma_final(self, G64, signs, Psi64):
        Psi = torch.empty(self.D, self.k, dtype=torch.float32, device=self.device)
        Gm = torch.empty(self.n_p, self.k, dtype=torch.float32, device=self.device)
        sg = np.ascontiguousarray(signs, np.int32)
        check(lib().tpo_shard_gamma_final(self._p(G64), self.n_p, self.k, sg.ctypes.data_as(C.c_void_p),
                                          self._p(Psi64), self.D, self._p(Psi), self._p(Gm), *self._ws(), self._st()))
        return Psi, Gm

    def onmf_init(self, Gamma_p, Psi, sigma):
        U, H = self._z(self.n_p, self.k), self._z(self.D, self.k)
        sig = np.ascontiguousarray(sigma, np.float64)
        check(lib().tpo_shard_onmf_init(self._p(Gamma_p), self.n_p, self._p(Psi), sig.ctypes.data_as(C.c_void_p),
                                        self.D, self.k, self._p(U), self._p(H), *self._ws(), self._st()))
        return U, H

    def rtu(self, Rp, dinv, U):
        out = self._z(self.D, self.k)
        check(lib().tpo_shard_onmf_rtu(self._p(Rp), self._p(dinv), self._p(U), self.n_p, self.D, self.k,
                                       self._p(out), *self._ws(), self._st()))
        return out

    def h_update(self, H, RtU, UtU):
        check(lib().tpo_onmf_h_update(self._p(H), self._p(RtU), self._p(UtU), self.D, self.k, *self._ws(), self._st()))

    def rh(self, Rp, dinv, H):
        out = self._z(self.n_p, self.k)
        check(lib().tpo_shard_onmf_rh(self._p(Rp), self._p(dinv), self._p(H), self.n_p, self.D, self.k, self._p(out),
                                      self._st()))
        return out

    def u_update(self, U, RH, M):
        check(lib().tpo_shard_onmf_u_update(self._p(U), self._p(RH), self._p(M), self.n_p, self.k, self._st()))

    def nci_assign(self, U, Phi, labels):
        changed = torch.zeros(1, dtype=torch.int32, device=self.device)
        sums, counts = self._z(self.k, self.k), self._z(self.k)
        check(lib().tpo_shard_nci_assign(self._p(U), self._p(Phi), self.n_p, self.k, self._p(labels), self._p(changed),
                                         self._p(sums), self._p(counts), *self._ws(), self._st()))
        return changed, sums, counts

    def phi(self, sums, counts):
        Phi = self._z(self.k, self.k)
        check(lib().tpo_nci_phi(self._p(sums), self._p(counts), self.k, self._p(Phi), self._st()))
        return Phi

    def eye(self):
        return torch.eye(self.k, dtype=torch.float64, device=self.device)

    def labels(self):
        return torch.full((self.n_p,), -1, dtype=torch.int32, device=self.device)


def _sign_rule(s, a, vals, idxs):
    """R8 from the global column statistics: sum >= 0, else (near-zero sums) the sign of the
    largest-magnitude entry, the smallest global row index among equal magnitudes.  vals/idxs:
    per rank (world x k) signed value at the rank's argmax and its global row index."""
    k = s.shape[0]
    signs = np.ones(k, np.int32)
    for l in range(k):
        if abs(s[l]) < 1e-6 * a[l]:
            best, bi, bv = -1.0, None, 0.0
            for r in range(vals.shape[0]):
                m, i = abs(vals[r, l]), idxs[r, l]
                if m > best or (m == best and i < bi):
                    best, bi, bv = m, i, vals[r, l]
            signs[l] = -1 if bv < 0 else 1
        else:
            signs[l] = -1 if s[l] < 0 else 1
    return signs


def solve_sharded(ops, coll, Zhat_p, Q, row0: int, Tf: int = 5, Tg: int = 20):
    """a5-a9 on this rank's rows (features -> exact top-k -> ONMF -> NCI), the same steps as
    tpo_run with the fp64 partials all-reduced in between.  Returns (labels_p, Alg. 3 iterations)."""
    Rp, r = ops.features(Zhat_p, Q)
    coll.allreduce_sum(r)                                    # r = sum_i R'[i]
    dinv = ops.dinv(Rp, r)
    G = ops.gram(Rp, dinv)
    coll.allreduce_sum(G)                                    # G = R^T R
    Psi64, sigma = ops.eig(G, r)                             # replicated (identical G on every rank)
    G64 = ops.gamma(Rp, dinv, Psi64, sigma)
    k = sigma.shape[0]
    eye = torch.eye(k, dtype=torch.float64, device=G64.device)
    for p in range(3):                                       # CholeskyQR polish while ||G^T G - I|| > 1e-6
        g = ops.atb(G64, G64)
        coll.allreduce_sum(g)
        if float((g - eye).abs().max()) <= 1e-6 or p == 2:
            break
        ops.apply_chol(G64, g)
    s, a, v, i = ops.colstats(G64, row0)
    coll.allreduce_sum(s)
    coll.allreduce_sum(a)
    vals = coll.all_gather_rows(v)
    idxs = coll.all_gather_rows(i)
    signs = _sign_rule(s.cpu().numpy(), a.cpu().numpy(), vals.cpu().numpy(), idxs.cpu().numpy())
    Psi, Gamma_p = ops.gamma_final(G64, signs, Psi64)
    U, H = ops.onmf_init(Gamma_p, Psi, sigma)                # Alg. 2
    for t in range(Tf):
        RtU = ops.rtu(Rp, dinv, U)
        coll.allreduce_sum(RtU)
        UtU = ops.atb(U, U)
        coll.allreduce_sum(UtU)
        ops.h_update(H, RtU, UtU)
        RH = ops.rh(Rp, dinv, H)
        M = ops.atb(U, RH)
        coll.allreduce_sum(M)
        ops.u_update(U, RH, M)
    Phi = ops.eye()                                          # Alg. 3
    labels = ops.labels()
    iters = 0
    for t in range(Tg):
        changed, sums, counts = ops.nci_assign(U, Phi, labels)
        coll.allreduce_sum(changed)
        iters += 1
        if int(changed.item()) == 0 or t == Tg - 1:
            break
        coll.allreduce_sum(sums)
        coll.allreduce_sum(counts)
        Phi = ops.phi(sums, counts)
    return labels, iters
