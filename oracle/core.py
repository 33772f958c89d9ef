"""ctypes wrapper of oracle/tpo_oracle.c (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

Each wrapper widens/validates numpy inputs and returns numpy outputs.  The C functions
cite the paper passages they follow.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tpo_oracle.c")
_LIB = os.path.join(_HERE, "libtpo_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, IEEE semantics, OpenMP static schedules)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        i64, i32, dbl, vp = C.c_int64, C.c_int32, C.c_double, C.c_void_p
        L.oracle_degree_scales.argtypes = [i64, i64, vp, vp, vp, vp, vp]
        L.oracle_propagate.argtypes = [i64, i64, vp, vp, vp, vp, i64, dbl, i32, vp, vp]
        L.oracle_haar_q.argtypes = [i64, vp, vp]
        L.oracle_qr.argtypes = [i64, i64, vp, vp, vp]
        L.oracle_features.argtypes = [i64, i64, vp, vp, vp, vp, vp]
        L.oracle_affinity_matvec.argtypes = [i64, i64, vp, vp, vp, i64, vp]
        L.oracle_sym_eig.argtypes = [i64, vp, vp, vp]
        L.oracle_gram.argtypes = [i64, i64, vp, vp, vp]
        L.oracle_topk.argtypes = [i64, i64, vp, vp, i32, vp, vp, vp, vp]
        L.oracle_topk.restype = C.c_int
        L.oracle_topk_from_eig.argtypes = [i64, i64, vp, vp, i32, vp, vp, vp, vp, vp, vp]
        L.oracle_topk_from_eig.restype = C.c_int
        L.oracle_svd_reduce.argtypes = [i64, i64, vp, i64, vp, vp]
        L.oracle_svd_reduce_from_eig.argtypes = [i64, i64, vp, i64, vp, vp, vp, vp]
        L.oracle_onmf.argtypes = [i64, i64, i32, vp, vp, vp, vp, vp, i32, vp, vp]
        L.oracle_nci.argtypes = [i64, i32, vp, i32, vp, vp]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt)


def degree_scales(n, m, rowptr, col, val=None):
    rowptr, col, val = _c(rowptr, np.int64), _c(col, np.int32), _c(val, np.float32)
    su, sv = np.zeros(n), np.zeros(m)
    lib().oracle_degree_scales(n, m, _p(rowptr), _p(col), _p(val), _p(su), _p(sv))
    return su, sv


def propagate(n, m, rowptr, col, X, alpha, T, val=None):
    """(Z, Zhat) in fp64 from CSR(B) only (Eq. PX truncated at T hops; Eq. Z)."""
    rowptr, col, val = _c(rowptr, np.int64), _c(col, np.int32), _c(val, np.float32)
    X = _c(X, np.float32)
    d = X.shape[1]
    Z, Zh = np.zeros((n, d)), np.zeros((n, d))
    lib().oracle_propagate(n, m, _p(rowptr), _p(col), _p(val), _p(X), d, float(alpha), int(T), _p(Z), _p(Zh))
    return Z, Zh


def haar_q(G):
    G = _c(G, np.float64)
    d = G.shape[0]
    Q = np.zeros((d, d))
    lib().oracle_haar_q(d, _p(G), _p(Q))
    return Q


def qr(A):
    A = _c(A, np.float64)
    r, c = A.shape
    Q, R = np.zeros((r, c)), np.zeros((c, c))
    lib().oracle_qr(r, c, _p(A), _p(Q), _p(R))
    return Q, R


def features(Zhat, Q):
    """(R', dinv, r) in fp64 from fp32 Zhat and fp32 Q (Eqs. R-prime, Ri)."""
    Zhat, Q = _c(Zhat, np.float32), _c(Q, np.float32)
    n, d = Zhat.shape
    Rp, dinv, r = np.zeros((n, 2 * d)), np.zeros(n), np.zeros(2 * d)
    lib().oracle_features(n, d, _p(Zhat), _p(Q), _p(Rp), _p(dinv), _p(r))
    return Rp, dinv, r


def affinity_matvec(Rp, dinv, Y):
    Rp, dinv, Y = _c(Rp, np.float32), _c(dinv, np.float32), _c(Y, np.float64)
    n, D = Rp.shape
    b = Y.shape[1]
    out = np.zeros((n, b))
    lib().oracle_affinity_matvec(n, D, _p(Rp), _p(dinv), _p(Y), b, _p(out))
    return out


def sym_eig(A):
    A = _c(A, np.float64)
    D = A.shape[0]
    w, V = np.zeros(D), np.zeros((D, D))
    lib().oracle_sym_eig(D, _p(A), _p(w), _p(V))
    return w, V


def gram(Rp, dinv):
    """G = R^T R, R = diag(dinv) R' (step 1 of topk)."""
    Rp, dinv = _c(Rp, np.float32), _c(dinv, np.float32)
    n, D = Rp.shape
    G = np.zeros((D, D))
    lib().oracle_gram(n, D, _p(Rp), _p(dinv), _p(G))
    return G


def topk(Rp, dinv, k, eig="jacobi"):
    """Exact top-k singular triplets of R = diag(dinv) R' -> (Gamma, sigma, Psi, all eigenvalues of R^T R).
    eig="lapack" takes the eigenpairs of the D x D Gram from numpy.linalg.eigh (LAPACK, a library
    eigensolver; the oracle's own cyclic Jacobi is pinned against it) instead of the Jacobi sweeps,
    whose cost grows as D^3 per sweep -- for D = 2000 (small config)."""
    Rp, dinv = _c(Rp, np.float32), _c(dinv, np.float32)
    n, D = Rp.shape
    Gm, s, Ps, lam = np.zeros((n, k)), np.zeros(k), np.zeros((D, k)), np.zeros(D)
    if eig == "lapack":
        w, V = np.linalg.eigh(gram(Rp, dinv))
        w, V = np.ascontiguousarray(w), np.ascontiguousarray(V)
        rc = lib().oracle_topk_from_eig(n, D, _p(Rp), _p(dinv), int(k), _p(w), _p(V), _p(Gm), _p(s), _p(Ps),
                                        _p(lam))
    else:
        rc = lib().oracle_topk(n, D, _p(Rp), _p(dinv), int(k), _p(Gm), _p(s), _p(Ps), _p(lam))
    if rc != 0:
        raise ArithmeticError(f"oracle_topk rc={rc}")
    return Gm, s, Ps, lam


def svd_reduce(X, d, eig="jacobi"):
    """X' = Gamma Sigma of the exact top-d SVD of X (Eq. Xd), sign-fixed (R8); pass-through when
    d >= d_U.  Returns (X' n x d fp64, sigma (d,) or None on pass-through).  eig="lapack" takes the
    eigenpairs of X^T X from numpy.linalg.eigh (LAPACK) instead of the Jacobi sweeps."""
    X = _c(X, np.float32)
    n, dU = X.shape
    if d >= dU:
        Xr = np.zeros((n, dU))
        lib().oracle_svd_reduce(n, dU, _p(X), int(d), _p(Xr), None)
        return Xr, None
    Xr, s = np.zeros((n, d)), np.zeros(d)
    if eig == "lapack":
        w, V = np.linalg.eigh(gram(X, np.ones(n, np.float32)))
        w, V = np.ascontiguousarray(w), np.ascontiguousarray(V)
        lib().oracle_svd_reduce_from_eig(n, dU, _p(X), int(d), _p(w), _p(V), _p(Xr), _p(s))
    else:
        lib().oracle_svd_reduce(n, dU, _p(X), int(d), _p(Xr), _p(s))
    return Xr, s


def onmf(Rp, dinv, Gamma, sigma, Psi, Tf):
    Rp, dinv = _c(Rp, np.float32), _c(dinv, np.float32)
    Gamma, Psi, sigma = _c(Gamma, np.float32), _c(Psi, np.float32), _c(sigma, np.float64)
    n, D = Rp.shape
    k = Gamma.shape[1]
    U, H = np.zeros((n, k)), np.zeros((D, k))
    lib().oracle_onmf(n, D, k, _p(Rp), _p(dinv), _p(Gamma), _p(sigma), _p(Psi), int(Tf), _p(U), _p(H))
    return U, H


def nci(Ups, Tg):
    Ups = _c(Ups, np.float64)
    n, k = Ups.shape
    labels = np.zeros(n, np.int32)
    it = C.c_int32(0)
    lib().oracle_nci(n, k, _p(Ups), int(Tg), _p(labels), C.byref(it))
    return labels, int(it.value)


def cluster(Rp, dinv, Gamma, sigma, Psi, Tf, Tg):
    """Alg. 2 then Alg. 3 -> (labels, iterations of Alg. 3 used, Upsilon)."""
    U, _ = onmf(Rp, dinv, Gamma, sigma, Psi, Tf)
    labels, it = nci(U, Tg)
    return labels, it, U


def run(g, Tf=5, Tg=20, k=None):
    """Whole hot path on an ABG (synth.ABG): propagate -> Q -> features -> top-k -> cluster.
    Each stage's fp64 result is rounded to fp32 where the CUDA path stores fp32."""
    k = g.k if k is None else k
    Z, Zh = propagate(g.n, g.m, g.B_rowptr, g.B_col, g.X, g.alpha, g.T, g.B_val)
    Q = haar_q(g.G)
    Rp, dinv, r = features(Zh.astype(np.float32), Q.astype(np.float32))
    Rp32, dinv32 = Rp.astype(np.float32), dinv.astype(np.float32)
    Gm, s, Ps, lam = topk(Rp32, dinv32, k)
    labels, it, U = cluster(Rp32, dinv32, Gm.astype(np.float32), s, Ps.astype(np.float32), Tf, Tg)
    return dict(Z=Z, Zhat=Zh, Q=Q, Rp=Rp, dinv=dinv, r=r, Gamma=Gm, sigma=s, Psi=Ps, lam=lam,
                labels=labels, iters=it, Ups=U)
