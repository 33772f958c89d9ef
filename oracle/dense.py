"""Tiny-size dense definitions in numpy (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

These are the plain definitions written out densely -- usable only for small n -- and
serve to pin the C oracle:

* ``dense_L``            Eq. L as a dense matrix.
* ``series_Z``           Eq. PX as an explicit power series.
* ``neumann_Z``          Lemma 1's gamma -> infinity limit (1-alpha)(I - alpha L L^T)^{-1} X
                         (proof).
* ``msa_matrix``         Eq. s: the exact MSA matrix S.
* ``obj1``               Eq. obj1 for one partition.
* ``best_partition``     brute force over all partitions into <= k clusters (n <= 10).
* ``sin_theta``          robust sin of the largest principal angle.
* ``ari``                adjusted Rand index for label comparisons.
* ``halko_topk``         the randomised truncated SVD the paper cites for the top-k (Halko et
                         al., p = 10, q = 2 at SPEC.md:143), replayed
                         step by step with Householder QR (Halko mode).
"""
from __future__ import annotations

import math

import numpy as np


def dense_B(n, m, rowptr, col, val=None):
    B = np.zeros((n, m))
    for u in range(n):
        for e in range(rowptr[u], rowptr[u + 1]):
            B[u, col[e]] += 1.0 if val is None else float(val[e])
    return B


def dense_L(B):
    du, dv = B.sum(1), B.sum(0)
    su = np.where(du > 0, 1.0 / np.sqrt(np.where(du > 0, du, 1.0)), 0.0)
    sv = np.where(dv > 0, 1.0 / np.sqrt(np.where(dv > 0, dv, 1.0)), 0.0)
    return su[:, None] * B * sv[None, :]


def series_Z(L, X, alpha, T):
    """(1-alpha) sum_{r=0}^{T} alpha^r (L L^T)^r X, with the dense matrix power."""
    M = L @ L.T
    out = np.zeros_like(X, dtype=np.float64)
    P = np.eye(M.shape[0])
    c = (1.0 - alpha) if alpha < 1.0 else 1.0
    for r in range(T + 1):
        out += c * (alpha ** r) * (P @ X)
        P = P @ M
    return out


def neumann_Z(L, X, alpha):
    M = L @ L.T
    return (1.0 - alpha) * np.linalg.solve(np.eye(M.shape[0]) - alpha * M, X)


def rownorm(Z):
    nr = np.linalg.norm(Z, axis=1, keepdims=True)
    return np.where(nr > 0, Z / np.where(nr > 0, nr, 1.0), 0.0)


def msa_matrix(Zhat):
    """Eq. s: s(i,j) = e^{z_i.z_j} / (sqrt(sum_l e^{z_i.z_l}) sqrt(sum_l e^{z_j.z_l}))."""
    K = np.exp(Zhat @ Zhat.T)
    rs = K.sum(1)
    return K / np.sqrt(np.outer(rs, rs))


def obj1(S, labels):
    """Eq. obj1: sum_l (1/|C_l|) sum_{i in C_l, j not in C_l} s(u_i, u_j)."""
    labels = np.asarray(labels)
    tot = 0.0
    for c in np.unique(labels):
        inn = labels == c
        tot += S[np.ix_(inn, ~inn)].sum() / inn.sum()
    return tot


def partitions(n, k):
    """All set partitions of range(n) into at most k blocks (restricted-growth strings)."""
    a = [0] * n

    def rec(i, mx):
        if i == n:
            yield tuple(a)
            return
        for v in range(min(mx + 2, k)):
            a[i] = v
            yield from rec(i + 1, max(mx, v))

    if n == 0:
        yield ()
        return
    a[0] = 0
    yield from rec(1, 0)


def best_partition(S, k, exact_k=True):
    """Brute-force minimiser of Eq. obj1 over partitions into k (or <= k) non-empty blocks."""
    n = S.shape[0]
    best, arg, allv = math.inf, None, []
    for p in partitions(n, k):
        if exact_k and len(set(p)) != k:
            continue
        v = obj1(S, p)
        allv.append((v, p))
        if v < best:
            best, arg = v, p
    allv.sort()
    return arg, best, allv


def orth(A):
    q, _ = np.linalg.qr(np.asarray(A, dtype=np.float64))
    return q


def sin_theta(A, B):
    """Robust sin(max principal angle) between span(A) and span(B):
    ||Q_B - Q_A (Q_A^T Q_B)||_2 after fp64 Householder orthonormalisation."""
    qa, qb = orth(A), orth(B)
    return float(np.linalg.norm(qb - qa @ (qa.T @ qb), 2))


def ari(a, b):
    """Adjusted Rand index (Hubert & Arabie) from the contingency table."""
    a, b = np.asarray(a), np.asarray(b)
    ua, ia = np.unique(a, return_inverse=True)
    ub, ib = np.unique(b, return_inverse=True)
    ct = np.zeros((ua.size, ub.size), np.int64)
    np.add.at(ct, (ia, ib), 1)

    def c2(x):
        x = np.asarray(x, np.float64)
        return (x * (x - 1) / 2).sum()

    n = a.size
    s_ij, s_a, s_b = c2(ct), c2(ct.sum(1)), c2(ct.sum(0))
    tot = n * (n - 1) / 2
    exp = s_a * s_b / tot if tot > 0 else 0.0
    mx = 0.5 * (s_a + s_b)
    if mx == exp:
        return 1.0
    return float((s_ij - exp) / (mx - exp))


def contingency(a, b):
    a, b = np.asarray(a), np.asarray(b)
    ua, ia = np.unique(a, return_inverse=True)
    ub, ib = np.unique(b, return_inverse=True)
    ct = np.zeros((ua.size, ub.size), np.int64)
    np.add.at(ct, (ia, ib), 1)
    return ct


def nmi(a, b):
    """Normalised mutual information in the standard sqrt-normalised form
    sum n_ij log(n n_ij / (a_i b_j)) / sqrt(sum a_i log(a_i / n) * sum b_j log(b_j / n)) (reading R15:
    the printed numerator omits n inside the logarithm)."""
    ct = contingency(a, b).astype(np.float64)
    n = ct.sum()
    ra, rb = ct.sum(1), ct.sum(0)
    nz = ct > 0
    mi = (ct[nz] * np.log(n * ct[nz] / np.outer(ra, rb)[nz])).sum()
    ha, hb = (ra * np.log(ra / n)).sum(), (rb * np.log(rb / n)).sum()
    if ha == 0.0 or hb == 0.0:
        return 1.0 if ha == hb else 0.0
    return float(mi / np.sqrt(ha * hb))


def acc(pred, truth):
    """Clustering accuracy: the fraction of nodes whose predicted label maps to
    their true label under the best one-to-one mapping (Hungarian algorithm; scipy's
    linear_sum_assignment, a library primitive)."""
    from scipy.optimize import linear_sum_assignment
    ct = contingency(pred, truth)
    r, c = linear_sum_assignment(-ct)
    return float(ct[r, c].sum() / ct.sum())


def nci_objective(Rp, dinv, labels, k, Ups=None):
    """Lemma 4's quantities (Eq. obj5) by explicit construction: S~ = R R^T (n x n),
    Y the NCI matrix of labels; returns (Tr(Y^T S~ Y), Tr(Ups^T S~ Ups) or None)."""
    R = np.asarray(dinv, np.float64)[:, None] * np.asarray(Rp, np.float64)
    S = R @ R.T
    n = R.shape[0]
    Y = np.zeros((n, k))
    for l in range(k):
        idx = labels == l
        if idx.any():
            Y[idx, l] = 1.0 / np.sqrt(idx.sum())
    t1 = float(np.trace(Y.T @ S @ Y))
    t2 = None if Ups is None else float(np.trace(np.asarray(Ups).T @ S @ np.asarray(Ups)))
    return t1, t2


def sign_rule(Gm, Ps):
    """R8: flip each pair so that sum_i Gamma[i, l] >= 0; when |sum| < 1e-6 ||.||_1 use
    the sign of the largest-magnitude entry (smallest index among ties)."""
    Gm, Ps = Gm.copy(), Ps.copy()
    for l in range(Gm.shape[1]):
        s, a = Gm[:, l].sum(), np.abs(Gm[:, l]).sum()
        sg = (-1.0 if Gm[np.argmax(np.abs(Gm[:, l])), l] < 0 else 1.0) if abs(s) < 1e-6 * a else (-1.0 if s < 0 else 1.0)
        Gm[:, l] *= sg
        Ps[:, l] *= sg
    return Gm, Ps


def halko_topk(Rp, dinv, k, p, q, Omega):
    """Randomised truncated SVD of R = diag(dinv) R' (Halko, Martinsson and Tropp):
    Y = orth(R Omega) with Omega (D x (k+p)) given; q times Y = orth(R (R^T Y)); then the SVD
    Y^T R = U S V^T gives Gamma = Y U[:, :k], sigma = S[:k], Psi = V[:, :k]; sign rule R8.
    fp64 throughout, Householder QR (numpy/LAPACK) for orth.  Returns (Gamma, sigma, Psi)."""
    R = np.asarray(dinv, np.float64)[:, None] * np.asarray(Rp, np.float64)
    Y, _ = np.linalg.qr(R @ np.asarray(Omega, np.float64))
    for _ in range(q):
        Y, _ = np.linalg.qr(R @ (R.T @ Y))
    U, S, Vt = np.linalg.svd(Y.T @ R, full_matrices=False)
    Gm, Ps = sign_rule(Y @ U[:, :k], Vt[:k].T)
    return Gm, S[:k].copy(), Ps
