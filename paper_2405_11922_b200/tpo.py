"""Python binding of libtpo (include/tpo.h): argument marshalling only.

PyTorch provides device memory and streams; every step of the hot path runs in the CUDA
library.  Function names follow the C-ABI: propagate, haar_q, features, affinity_matvec,
topk_eig, cluster, run.  Tensors must be CUDA tensors of the documented dtype and be
contiguous; outputs are allocated here unless passed in.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from ._lib import CSR, TPO_EIG_EXACT, TPO_EIG_HALKO, check, lib  # noqa: F401


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _need(t, dtype, name, shape=None):
    if not (isinstance(t, torch.Tensor) and t.is_cuda):
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    return t


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


@dataclass
class DeviceGraph:
    """CSR(B) (n_u x n_v) and CSR(B^T) (n_v x n_u) of one ABG on the device."""
    n_u: int
    n_v: int
    nnz: int
    B_rowptr: torch.Tensor
    B_col: torch.Tensor
    Bt_rowptr: torch.Tensor
    Bt_col: torch.Tensor
    B_val: Optional[torch.Tensor] = None
    Bt_val: Optional[torch.Tensor] = None

    def csr(self):
        B = CSR(self.n_u, self.n_v, self.nnz, self.B_rowptr.data_ptr(), self.B_col.data_ptr(),
                None if self.B_val is None else self.B_val.data_ptr())
        Bt = CSR(self.n_v, self.n_u, self.nnz, self.Bt_rowptr.data_ptr(), self.Bt_col.data_ptr(),
                 None if self.Bt_val is None else self.Bt_val.data_ptr())
        return B, Bt

    def target(self, side: str = "U") -> "DeviceGraph":
        """The graph oriented for clustering `side`: U as given, or V (the roles of B
        and B^T swap, X is then X_V).  No copy: the same device CSRs."""
        if side == "U":
            return self
        if side != "V":
            raise ValueError("target side must be 'U' or 'V'")
        return DeviceGraph(self.n_v, self.n_u, self.nnz, self.Bt_rowptr, self.Bt_col, self.B_rowptr, self.B_col,
                           self.Bt_val, self.B_val)


def to_device_graph(n_u, n_v, B_rowptr, B_col, Bt_rowptr, Bt_col, B_val=None, Bt_val=None,
                    device="cuda", non_blocking=False) -> DeviceGraph:
    def dev(a, dt):
        if a is None:
            return None
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
        return t.to(device=device, dtype=dt, non_blocking=non_blocking).contiguous()
    return DeviceGraph(int(n_u), int(n_v), int(len(B_col)), dev(B_rowptr, torch.int64), dev(B_col, torch.int32),
                       dev(Bt_rowptr, torch.int64), dev(Bt_col, torch.int32),
                       dev(B_val, torch.float32), dev(Bt_val, torch.float32))


def propagate(g: DeviceGraph, X: torch.Tensor, alpha: float, T: int, Z=None, Zhat=None, want_zhat=True,
              stream=None):
    """a1-a3 (tpo_propagate): returns (Z, Zhat)."""
    n, d = X.shape
    _need(X, torch.float32, "X", (g.n_u, d))
    Z = torch.empty_like(X) if Z is None else _need(Z, torch.float32, "Z", X.shape)
    if want_zhat:
        Zhat = torch.empty_like(X) if Zhat is None else _need(Zhat, torch.float32, "Zhat", X.shape)
    else:
        Zhat = None
    L = lib()
    nbytes = L.tpo_propagate_ws(g.n_u, g.n_v, g.nnz, d)
    ws = _ws(nbytes, X.device)
    B, Bt = g.csr()
    check(L.tpo_propagate(C.byref(B), C.byref(Bt), _ptr(X), d, float(alpha), int(T), _ptr(Z), _ptr(Zhat),
                          _ptr(ws), ws.numel(), _stream(stream)))
    return Z, Zhat


def haar_q(G: np.ndarray) -> np.ndarray:
    """a4 (tpo_haar_q, host): Q of the positive-diagonal QR of the Gaussian G."""
    G = np.ascontiguousarray(G, dtype=np.float64)
    d = G.shape[0]
    Q = np.empty((d, d), np.float64)
    check(lib().tpo_haar_q(G.ctypes.data_as(C.c_void_p), d, Q.ctypes.data_as(C.c_void_p)))
    return Q


def haar_q_dev(G: np.ndarray, device="cuda", stream=None) -> torch.Tensor:
    """a4 on the device (tpo_haar_q_dev): fp32 Q of the positive-diagonal QR of G."""
    G = np.ascontiguousarray(G, dtype=np.float64)
    d = G.shape[0]
    Q = torch.empty((d, d), dtype=torch.float32, device=device)
    L = lib()
    ws = _ws(L.tpo_haar_q_dev_ws(d), Q.device)
    check(L.tpo_haar_q_dev(G.ctypes.data_as(C.c_void_p), d, _ptr(Q), _ptr(ws), ws.numel(), _stream(stream)))
    return Q


def features(Zhat: torch.Tensor, Q: torch.Tensor, Rp=None, dinv=None, want_r=False, stream=None):
    """a5 (tpo_features): returns (Rp, dinv, r or None)."""
    n, d = Zhat.shape
    _need(Zhat, torch.float32, "Zhat")
    _need(Q, torch.float32, "Q", (d, d))
    Rp = torch.empty((n, 2 * d), dtype=torch.float32, device=Zhat.device) if Rp is None else Rp
    dinv = torch.empty(n, dtype=torch.float32, device=Zhat.device) if dinv is None else dinv
    r = torch.empty(2 * d, dtype=torch.float64, device=Zhat.device) if want_r else None
    L = lib()
    ws = _ws(L.tpo_features_ws(n, d), Zhat.device)
    check(L.tpo_features(_ptr(Zhat), n, d, _ptr(Q), _ptr(Rp), _ptr(dinv), _ptr(r), _ptr(ws), ws.numel(),
                         _stream(stream)))
    return Rp, dinv, r


def affinity_matvec(Rp: torch.Tensor, dinv: torch.Tensor, Y: torch.Tensor, out=None, stream=None):
    """a6 (tpo_affinity_matvec): dinv . R'(R'^T (dinv . Y))."""
    n, D = Rp.shape
    _need(Rp, torch.float32, "Rp")
    _need(dinv, torch.float32, "dinv", (n,))
    _need(Y, torch.float32, "Y")
    b = Y.shape[1]
    out = torch.empty_like(Y) if out is None else out
    L = lib()
    ws = _ws(L.tpo_affinity_matvec_ws(n, D, b), Rp.device)
    check(L.tpo_affinity_matvec(_ptr(Rp), _ptr(dinv), n, D, _ptr(Y), b, _ptr(out), _ptr(ws), ws.numel(),
                                _stream(stream)))
    return out


def rowgemm_f64(A: torch.Tensor, W: torch.Tensor, rs=None, out=None, stream=None):
    """tpo_rowgemm_f64: out = diag(rs) A W in fp64 (A n x K fp32, W K x N fp64)."""
    n, K = A.shape
    _need(A, torch.float32, "A")
    _need(W, torch.float64, "W")
    N = W.shape[1]
    if rs is not None:
        _need(rs, torch.float32, "rs", (n,))
    out = torch.empty(n, N, dtype=torch.float64, device=A.device) if out is None else out
    L = lib()
    ws = _ws(L.tpo_rowgemm_f64_ws(n, K, N), A.device)
    check(L.tpo_rowgemm_f64(_ptr(A), n, K, _ptr(rs) if rs is not None else None, _ptr(W), N, _ptr(out), _ptr(ws),
                            ws.numel(), _stream(stream)))
    return out


def onmf_rtu(Rp: torch.Tensor, dinv: torch.Tensor, U: torch.Tensor, out=None, stream=None):
    """tpo_shard_onmf_rtu over all rows: RtU = R'^T (dinv . U) (D x k fp64; Alg. 2's R^T Ups)."""
    n, D = Rp.shape
    _need(Rp, torch.float32, "Rp")
    _need(dinv, torch.float32, "dinv", (n,))
    _need(U, torch.float64, "U")
    k = U.shape[1]
    out = torch.empty(D, k, dtype=torch.float64, device=Rp.device) if out is None else out
    L = lib()
    ws = _ws(L.tpo_shard_solver_ws(n, D // 2, k), Rp.device)
    check(L.tpo_shard_onmf_rtu(_ptr(Rp), _ptr(dinv), _ptr(U), n, D, k, _ptr(out), _ptr(ws), ws.numel(),
                               _stream(stream)))
    return out


def affinity_matvec_rfree(Zhat: torch.Tensor, Q: torch.Tensor, Y: torch.Tensor, chunk_rows: int = 0, out=None,
                          stream=None):
    """a6 without materialising R' (tpo_affinity_matvec_rfree): R' rows recomputed from Zhat in chunks."""
    n, d = Zhat.shape
    _need(Zhat, torch.float32, "Zhat")
    _need(Q, torch.float32, "Q", (d, d))
    _need(Y, torch.float32, "Y")
    b = Y.shape[1]
    out = torch.empty_like(Y) if out is None else out
    L = lib()
    ws = _ws(L.tpo_affinity_matvec_rfree_ws(n, d, b, int(chunk_rows)), Zhat.device)
    check(L.tpo_affinity_matvec_rfree(_ptr(Zhat), n, d, _ptr(Q), _ptr(Y), b, _ptr(out), int(chunk_rows), _ptr(ws),
                                      ws.numel(), _stream(stream)))
    return out


def gram(Rp: torch.Tensor, dinv: torch.Tensor, stream=None) -> torch.Tensor:
    """a7 step 1 (tpo_gram): G = R'^T diag(dinv^2) R' as a D x D fp64 tensor."""
    n, D = Rp.shape
    _need(Rp, torch.float32, "Rp")
    _need(dinv, torch.float32, "dinv", (n,))
    G = torch.empty((D, D), dtype=torch.float64, device=Rp.device)
    L = lib()
    ws = _ws(L.tpo_gram_ws(n, D), Rp.device)
    check(L.tpo_gram(_ptr(Rp), _ptr(dinv), n, D, _ptr(G), _ptr(ws), ws.numel(), _stream(stream)))
    return G


def topk_eig(Rp: torch.Tensor, dinv: torch.Tensor, k: int, mode: int = TPO_EIG_EXACT, p: int = 10, q: int = 2,
             Omega: Optional[torch.Tensor] = None, stream=None):
    """a7 (tpo_topk_eig): returns (Gamma [n,k] fp32, sigma np.float64[k], Psi [D,k] fp32)."""
    n, D = Rp.shape
    _need(Rp, torch.float32, "Rp")
    _need(dinv, torch.float32, "dinv", (n,))
    if mode == TPO_EIG_HALKO:
        _need(Omega, torch.float32, "Omega", (D, k + p))
    Gamma = torch.empty((n, k), dtype=torch.float32, device=Rp.device)
    Psi = torch.empty((D, k), dtype=torch.float32, device=Rp.device)
    sigma = np.zeros(k, np.float64)
    L = lib()
    ws = _ws(L.tpo_topk_eig_ws(n, D, k, mode, p), Rp.device)
    check(L.tpo_topk_eig(_ptr(Rp), _ptr(dinv), n, D, int(k), int(mode), int(p), int(q), _ptr(Omega), _ptr(Gamma),
                         sigma.ctypes.data_as(C.c_void_p), _ptr(Psi), _ptr(ws), ws.numel(), _stream(stream)))
    return Gamma, sigma, Psi


def svd_reduce(X: torch.Tensor, d: int, out=None, stream=None):
    """Sec. 3.2.1 (tpo_svd_reduce): X' = Gamma Sigma of the exact top-d SVD of X (Eq. Xd), sign-fixed;
    returns (X' [n, d] fp32, sigma np.float64[d] or None on pass-through d == d_u)."""
    n, du = X.shape
    _need(X, torch.float32, "X")
    d = int(d)
    out = torch.empty((n, du if d >= du else d), dtype=torch.float32, device=X.device) if out is None else out
    sigma = np.zeros(max(d, 1), np.float64)
    L = lib()
    ws = _ws(L.tpo_svd_reduce_ws(n, du, d), X.device)
    check(L.tpo_svd_reduce(_ptr(X), n, du, d, _ptr(out), sigma.ctypes.data_as(C.c_void_p), _ptr(ws), ws.numel(),
                           _stream(stream)))
    return out, (None if d >= du else sigma[:d])


def evaluate(pred: torch.Tensor, truth: torch.Tensor, k_pred: int, k_true: int, stream=None) -> dict:
    """Clustering metrics (tpo_eval): {'ari', 'nmi', 'acc'} of pred vs truth."""
    _need(pred, torch.int32, "pred")
    _need(truth, torch.int32, "truth", pred.shape)
    m = np.zeros(3, np.float64)
    L = lib()
    ws = _ws(L.tpo_eval_ws(int(k_pred), int(k_true)), pred.device)
    check(L.tpo_eval(_ptr(pred), _ptr(truth), pred.numel(), int(k_pred), int(k_true), m.ctypes.data_as(C.c_void_p),
                     _ptr(ws), ws.numel(), _stream(stream)))
    return {"ari": float(m[0]), "nmi": float(m[1]), "acc": float(m[2])}


def objective(Rp: torch.Tensor, dinv: torch.Tensor, labels: torch.Tensor, k: int, Ups: Optional[torch.Tensor] = None,
              stream=None):
    """Lemma 4 monitor (tpo_objective): (||R^T Y||_F^2, ||R^T Ups||_F^2 or None) for the NCI Y of labels."""
    n, D = Rp.shape
    _need(Rp, torch.float32, "Rp")
    _need(dinv, torch.float32, "dinv", (n,))
    _need(labels, torch.int32, "labels", (n,))
    if Ups is not None:
        _need(Ups, torch.float64, "Ups", (n, k))
    out = np.zeros(2, np.float64)
    L = lib()
    ws = _ws(L.tpo_objective_ws(n, D, int(k)), Rp.device)
    check(L.tpo_objective(_ptr(Rp), _ptr(dinv), n, D, int(k), _ptr(labels), _ptr(Ups), out.ctypes.data_as(C.c_void_p),
                          _ptr(ws), ws.numel(), _stream(stream)))
    return float(out[0]), (float(out[1]) if Ups is not None else None)


def cluster(Rp: torch.Tensor, dinv: torch.Tensor, Gamma: torch.Tensor, sigma: np.ndarray, Psi: torch.Tensor,
            Tf: int = 5, Tg: int = 20, labels=None, stream=None):
    """a8-a9 (tpo_cluster): returns (labels int32 [n], iterations of Alg. 3 run)."""
    n, D = Rp.shape
    k = Gamma.shape[1]
    _need(Rp, torch.float32, "Rp")
    _need(dinv, torch.float32, "dinv", (n,))
    _need(Gamma, torch.float32, "Gamma", (n, k))
    _need(Psi, torch.float32, "Psi", (D, k))
    sigma = np.ascontiguousarray(sigma, dtype=np.float64)
    labels = torch.empty(n, dtype=torch.int32, device=Rp.device) if labels is None else labels
    it = C.c_int32(0)
    L = lib()
    ws = _ws(L.tpo_cluster_ws(n, D, k), Rp.device)
    check(L.tpo_cluster(_ptr(Rp), _ptr(dinv), n, D, int(k), _ptr(Gamma), sigma.ctypes.data_as(C.c_void_p), _ptr(Psi),
                        int(Tf), int(Tg), _ptr(labels), C.byref(it), _ptr(ws), ws.numel(), _stream(stream)))
    return labels, int(it.value)


def topk_eig_rfree(Zhat: torch.Tensor, Q: torch.Tensor, k: int, chunk_rows: int = 0, stream=None):
    """a7 without materialising R' (tpo_topk_eig_rfree, exact mode): returns (Gamma [n,k] fp32,
    sigma np.float64[k], Psi [2d,k] fp32, dinv [n] fp32)."""
    n, d = Zhat.shape
    _need(Zhat, torch.float32, "Zhat")
    _need(Q, torch.float32, "Q", (d, d))
    Gamma = torch.empty((n, k), dtype=torch.float32, device=Zhat.device)
    Psi = torch.empty((2 * d, k), dtype=torch.float32, device=Zhat.device)
    dinv = torch.empty(n, dtype=torch.float32, device=Zhat.device)
    sigma = np.zeros(k, np.float64)
    L = lib()
    ws = _ws(L.tpo_topk_eig_rfree_ws(n, d, int(k), int(chunk_rows)), Zhat.device)
    check(L.tpo_topk_eig_rfree(_ptr(Zhat), n, d, _ptr(Q), int(k), _ptr(Gamma), sigma.ctypes.data_as(C.c_void_p),
                               _ptr(Psi), _ptr(dinv), int(chunk_rows), _ptr(ws), ws.numel(), _stream(stream)))
    return Gamma, sigma, Psi, dinv


def cluster_rfree(Zhat: torch.Tensor, Q: torch.Tensor, dinv: torch.Tensor, Gamma: torch.Tensor, sigma: np.ndarray,
                  Psi: torch.Tensor, Tf: int = 5, Tg: int = 20, chunk_rows: int = 0, labels=None, stream=None):
    """a8-a9 without materialising R' (tpo_cluster_rfree): returns (labels int32 [n], Alg. 3 iterations)."""
    n, d = Zhat.shape
    k = Gamma.shape[1]
    _need(Zhat, torch.float32, "Zhat")
    _need(Q, torch.float32, "Q", (d, d))
    _need(dinv, torch.float32, "dinv", (n,))
    _need(Gamma, torch.float32, "Gamma", (n, k))
    _need(Psi, torch.float32, "Psi", (2 * d, k))
    sigma = np.ascontiguousarray(sigma, dtype=np.float64)
    labels = torch.empty(n, dtype=torch.int32, device=Zhat.device) if labels is None else labels
    it = C.c_int32(0)
    L = lib()
    ws = _ws(L.tpo_cluster_rfree_ws(n, d, int(k), int(chunk_rows)), Zhat.device)
    check(L.tpo_cluster_rfree(_ptr(Zhat), n, d, _ptr(Q), _ptr(dinv), int(k), _ptr(Gamma),
                              sigma.ctypes.data_as(C.c_void_p), _ptr(Psi), int(Tf), int(Tg), _ptr(labels), C.byref(it),
                              int(chunk_rows), _ptr(ws), ws.numel(), _stream(stream)))
    return labels, int(it.value)


class Runner:
    """Whole hot path (tpo_run) with a workspace kept across calls."""

    def __init__(self, g: DeviceGraph, d: int, k: int, mode: int = TPO_EIG_EXACT, p: int = 10, device="cuda"):
        self.g, self.d, self.k, self.mode, self.p = g, d, k, mode, p
        self.ws = _ws(lib().tpo_run_ws(g.n_u, g.n_v, g.nnz, d, k, mode, p), device)
        self.labels = torch.empty(g.n_u, dtype=torch.int32, device=device)
        self.timings = np.zeros(4, np.float64)

    def __call__(self, X: torch.Tensor, alpha: float, T: int, G, Tf: int = 5, Tg: int = 20,
                 q: int = 2, Omega: Optional[torch.Tensor] = None, stream=None):
        """G: the d x d fp64 Gaussian of Alg. 1 L6, a device tensor (numpy arrays are uploaded)."""
        _need(X, torch.float32, "X", (self.g.n_u, self.d))
        if not isinstance(G, torch.Tensor):
            G = torch.from_numpy(np.ascontiguousarray(G, dtype=np.float64)).to(X.device)
        _need(G, torch.float64, "G", (self.d, self.d))
        B, Bt = self.g.csr()
        check(lib().tpo_run(C.byref(B), C.byref(Bt), _ptr(X), self.d, float(alpha), int(T), int(self.k),
                            _ptr(G), int(self.mode), _ptr(Omega), int(self.p), int(q), int(Tf),
                            int(Tg), _ptr(self.labels), self.timings.ctypes.data_as(C.c_void_p), _ptr(self.ws),
                            self.ws.numel(), _stream(stream)))
        return self.labels


def _host(t, dtype, name, shape):
    """A contiguous CPU tensor of `dtype` and `shape` (numpy arrays are wrapped, not copied)."""
    if isinstance(t, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(t))
    if not isinstance(t, torch.Tensor) or t.is_cuda:
        raise TypeError(f"{name} must be a host (CPU) tensor or numpy array")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous() or tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must be contiguous with shape {tuple(shape)}, got {tuple(t.shape)}")
    return t


class HostRunner:
    """Whole hot path from HOST inputs (tpo_run_host): the inputs are copied inside the call,
    the Haar QR of G runs beside their copies, the labels come back to a host array.  Pinned
    host tensors make the copies asynchronous."""

    def __init__(self, n_u: int, n_v: int, nnz: int, d: int, k: int, weighted: bool = False,
                 mode: int = TPO_EIG_EXACT, p: int = 10, device="cuda"):
        self.n_u, self.n_v, self.nnz, self.d, self.k = n_u, n_v, nnz, d, k
        self.weighted, self.mode, self.p = weighted, mode, p
        self.ws = _ws(lib().tpo_run_host_ws(n_u, n_v, nnz, d, k, mode, p, int(weighted)), device)
        self.timings = np.zeros(4, np.float64)

    def __call__(self, B_rowptr, B_col, Bt_rowptr, Bt_col, X, G, alpha: float, T: int, Tf: int = 5, Tg: int = 20,
                 B_val=None, Bt_val=None, labels=None, q: int = 2, Omega: Optional[torch.Tensor] = None, stream=None):
        n, m, e, d = self.n_u, self.n_v, self.nnz, self.d
        brp = _host(B_rowptr, torch.int64, "B_rowptr", (n + 1,))
        bci = _host(B_col, torch.int32, "B_col", (e,))
        trp = _host(Bt_rowptr, torch.int64, "Bt_rowptr", (m + 1,))
        tci = _host(Bt_col, torch.int32, "Bt_col", (e,))
        Xh = _host(X, torch.float32, "X", (n, d))
        Gh = _host(G, torch.float64, "G", (d, d))
        if (B_val is None) != (not self.weighted) or (Bt_val is None) != (not self.weighted):
            raise ValueError("weights must be given for both B and Bt exactly when the runner is weighted")
        bv = None if B_val is None else _host(B_val, torch.float32, "B_val", (e,))
        tv = None if Bt_val is None else _host(Bt_val, torch.float32, "Bt_val", (e,))
        if labels is None:
            labels = torch.empty(n, dtype=torch.int32)
        labels = _host(labels, torch.int32, "labels", (n,))
        B = CSR(n, m, e, brp.data_ptr(), bci.data_ptr(), None if bv is None else bv.data_ptr())
        Bt = CSR(m, n, e, trp.data_ptr(), tci.data_ptr(), None if tv is None else tv.data_ptr())
        check(lib().tpo_run_host(C.byref(B), C.byref(Bt), C.c_void_p(Xh.data_ptr()), d, float(alpha), int(T),
                                 int(self.k), C.c_void_p(Gh.data_ptr()), int(self.mode), _ptr(Omega), int(self.p),
                                 int(q), int(Tf), int(Tg), C.c_void_p(labels.data_ptr()),
                                 self.timings.ctypes.data_as(C.c_void_p), _ptr(self.ws), self.ws.numel(),
                                 _stream(stream)))
        return labels


def run(g: DeviceGraph, X: torch.Tensor, alpha: float, T: int, k: int, G: np.ndarray, mode=TPO_EIG_EXACT,
        Tf=5, Tg=20, p=10, q=2, Omega=None):
    """Whole hot path (tpo_run): returns (labels, timings_ms[4])."""
    r = Runner(g, X.shape[1], k, mode, p, X.device)
    labels = r(X, alpha, T, G, Tf, Tg, q, Omega)
    return labels, r.timings.copy()
