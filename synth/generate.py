"""Seeded planted-cluster ABG generator (BASELINE.json "configs").

Everything here is input drawing: degrees, endpoints, attribute rows, and the i.i.d.
Gaussian matrices that the method consumes as inputs (G of Alg. 1 L6, PAPER.md:481,
and Omega, the Gaussian test matrix of the randomised SVD cited at PAPER.md:574).
None of the method's arithmetic lives here.

Independent random streams come from numpy's PCG64 seeded with (seed, purpose).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_PURPOSE = {"graph": 1, "X": 2, "G": 3, "Omega": 4, "perm": 5, "aux": 6}


def _rng(seed: int, purpose: str) -> np.random.Generator:
    return np.random.default_rng([int(seed), _PURPOSE[purpose]])


# BASELINE.json configs[0..4] with the SURVEY.md §8(d) readings.
CONFIGS = {
    "tiny": dict(n=2_000, m=3_000, k=5, d=300, alpha=0.5, T=3,
                 deg=("poisson", 8.0), p_in=0.80, pop=("uniform",),
                 x=("sparse_sig", 0.05, 0.15, 30)),
    "small": dict(n=50_000, m=80_000, k=10, d=1000, alpha=0.5, T=5,
                  deg=("poisson", 20.0), p_in=0.70, pop=("zipf", 1.1),
                  x=("sparse_sig", 0.01, 0.03, 100)),
    "medium": dict(n=500_000, m=300_000, k=20, d=256, alpha=0.6, T=5,
                   deg=("zipf", 1.2, 222), p_in=0.60, pop=("zipf", 1.2),
                   x=("gaussian", 1.0)),
    "large": dict(n=2_000_000, m=1_000_000, k=50, d=128, alpha=0.5, T=8,
                  deg=("zipf", 1.3, 450), p_in=0.50, pop=("zipf", 1.3),
                  x=("gaussian", 1.0)),
    "xl": dict(n=10_000_000, m=4_000_000, k=100, d=128, alpha=0.5, T=10,
               deg=("zipf", 1.3, 450), p_in=0.50, pop=("zipf", 1.3),
               x=("gaussian", 1.0)),
}


@dataclass
class ABG:
    """CSR(B) (n x m) and CSR(B^T) (m x n) of one graph, plus X, G, Omega and planted labels."""
    n: int
    m: int
    d: int
    k: int
    alpha: float
    T: int
    B_rowptr: np.ndarray      # int64 [n+1]
    B_col: np.ndarray         # int32 [E], strictly increasing within a row
    Bt_rowptr: np.ndarray     # int64 [m+1]
    Bt_col: np.ndarray        # int32 [E]
    X: np.ndarray             # float32 [n, d], rows L2-normalised by the generator
    G: np.ndarray             # float64 [d, d], i.i.d. N(0,1)
    Omega: np.ndarray         # float32 [2d, k+p], i.i.d. N(0,1)
    truth: np.ndarray         # int32 [n] planted cluster of each U node
    B_val: Optional[np.ndarray] = None   # float32 [E] or None (unit weights)
    Bt_val: Optional[np.ndarray] = None
    name: str = "custom"
    seed: int = 0
    extra: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.B_col.shape[0])

    def stats(self) -> dict:
        du = np.diff(self.B_rowptr)
        dv = np.diff(self.Bt_rowptr)
        return dict(n=self.n, m=self.m, nnz=self.nnz, d=self.d, k=self.k,
                    max_deg_u=int(du.max(initial=0)), median_deg_u=float(np.median(du)) if du.size else 0.0,
                    max_deg_v=int(dv.max(initial=0)), median_deg_v=float(np.median(dv)) if dv.size else 0.0,
                    isolated_u=int((du == 0).sum()), isolated_v=int((dv == 0).sum()))


def csr_from_edges(u: np.ndarray, v: np.ndarray, n: int, m: int, w: Optional[np.ndarray] = None):
    """CSR of B (rows u) and of B^T (rows v) from a duplicate-free edge list, by stable sorts."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    if w is None:
        kb = np.sort(u * m + v)
        kt = np.sort(v * n + u)
        B_col = (kb % m).astype(np.int32)
        Bt_col = (kt % n).astype(np.int32)
        B_rowptr = np.zeros(n + 1, np.int64)
        np.cumsum(np.bincount(kb // m, minlength=n), out=B_rowptr[1:])
        Bt_rowptr = np.zeros(m + 1, np.int64)
        np.cumsum(np.bincount(kt // n, minlength=m), out=Bt_rowptr[1:])
        return B_rowptr, B_col, Bt_rowptr, Bt_col, None, None
    w = np.asarray(w, dtype=np.float32)
    ob = np.lexsort((v, u))
    ot = np.lexsort((u, v))
    B_rowptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(u, minlength=n), out=B_rowptr[1:])
    Bt_rowptr = np.zeros(m + 1, np.int64)
    np.cumsum(np.bincount(v, minlength=m), out=Bt_rowptr[1:])
    return (B_rowptr, v[ob].astype(np.int32), Bt_rowptr, u[ot].astype(np.int32),
            np.ascontiguousarray(w[ob]), np.ascontiguousarray(w[ot]))


def _zipf_cdf(N: int, s: float) -> np.ndarray:
    x = np.arange(1, N + 1, dtype=np.float64)
    p = x ** (-s)
    c = np.cumsum(p)
    return c / c[-1]


def _draw_degrees(rng, n, deg):
    if deg[0] == "poisson":
        return rng.poisson(deg[1], size=n).astype(np.int64)
    if deg[0] == "zipf":       # truncated Zipf(s) on [1, xmax] (SURVEY.md A.3 caps)
        cdf = _zipf_cdf(int(deg[2]), float(deg[1]))
        return (np.searchsorted(cdf, rng.random(n), side="right") + 1).astype(np.int64)
    if deg[0] == "const":
        return np.full(n, int(deg[1]), np.int64)
    raise ValueError(deg)


def _draw_endpoints(rng, ucl, k, S, p_in, pop):
    """Planted V index for each edge: own block w.p. p_in else a uniform other block;
    position in the block uniform or by rank-Zipf popularity (ranks are shuffled later
    by the global V permutation)."""
    E = ucl.shape[0]
    intra = rng.random(E) < p_in
    if k > 1:
        other = (ucl + 1 + rng.integers(0, k - 1, size=E)) % k
        blk = np.where(intra, ucl, other)
    else:
        blk = ucl.copy()
    if pop[0] == "uniform":
        pos = rng.integers(0, S, size=E)
    else:
        cdf = _zipf_cdf(S, float(pop[1]))
        pos = np.minimum(np.searchsorted(cdf, rng.random(E), side="right"), S - 1)
    return blk.astype(np.int64) * S + pos.astype(np.int64)


def _dedup_edges(rng, u_pl, v_pl, ucl, k, S, m, p_in, pop, max_rounds=200):
    """Per-row duplicate-free sampling: redraw duplicated (u, v) pairs until none remain."""
    keys = np.sort(u_pl * m + v_pl)
    dup = np.zeros(keys.shape[0], bool)
    dup[1:] = keys[1:] == keys[:-1]
    base = keys[~dup]
    pend_u = (keys[dup] // m).astype(np.int64)
    extra = np.empty(0, np.int64)
    for _ in range(max_rounds):
        if pend_u.size == 0:
            break
        cand = pend_u * m + _draw_endpoints(rng, ucl[pend_u], k, S, p_in, pop)
        order = np.argsort(cand, kind="stable")
        cs = cand[order]
        first = np.ones(cs.shape[0], bool)
        first[1:] = cs[1:] != cs[:-1]
        i0 = np.searchsorted(base, cs)
        in_base = (i0 < base.shape[0]) & (base[np.minimum(i0, base.shape[0] - 1)] == cs)
        if extra.size:
            i1 = np.searchsorted(extra, cs)
            in_extra = (i1 < extra.shape[0]) & (extra[np.minimum(i1, extra.shape[0] - 1)] == cs)
        else:
            in_extra = np.zeros(cs.shape[0], bool)
        ok = first & ~in_base & ~in_extra
        extra = np.sort(np.concatenate([extra, cs[ok]]))
        pend_u = cs[~ok] // m
    allk = np.sort(np.concatenate([base, extra])) if extra.size else base
    return allk // m, allk % m


def _draw_X(rng, n, d, k, cl, xm):
    if xm[0] == "sparse_sig":     # base mask + per-cluster signature columns (x3 values)
        p_base, p_sig, width = float(xm[1]), float(xm[2]), int(xm[3])
        X = np.zeros((n, d), np.float32)
        chunk = 1 << 16
        for s in range(0, n, chunk):
            e = min(n, s + chunk)
            mask = rng.random((e - s, d), dtype=np.float32) < p_base
            val = rng.random((e - s, d), dtype=np.float32)
            Xc = np.where(mask, val, np.float32(0))
            cols = (cl[s:e, None] * width + np.arange(width)[None, :]) % d
            smask = rng.random((e - s, width), dtype=np.float32) < p_sig
            sval = np.float32(3.0) * rng.random((e - s, width), dtype=np.float32)
            rows = np.repeat(np.arange(e - s), width).reshape(e - s, width)
            cur = Xc[rows, cols]
            Xc[rows, cols] = np.where(smask, sval, cur)
            X[s:e] = Xc
    elif xm[0] == "gaussian":     # planted Gaussian cluster means plus unit noise
        sigma = float(xm[1])
        mu = rng.standard_normal((k, d), dtype=np.float32) * np.float32(sigma)
        X = np.empty((n, d), np.float32)
        chunk = 1 << 18
        for s in range(0, n, chunk):
            e = min(n, s + chunk)
            X[s:e] = mu[cl[s:e]] + rng.standard_normal((e - s, d), dtype=np.float32)
    elif xm[0] == "uniform":
        X = rng.random((n, d), dtype=np.float32)
    else:
        raise ValueError(xm)
    nrm = np.sqrt(np.einsum("ij,ij->i", X, X, dtype=np.float64)).astype(np.float32)
    nz = nrm > 0
    X[nz] /= nrm[nz, None]
    return X


def planted_abg(n: int, m: int, k: int, d: int, *, deg=("poisson", 8.0), p_in=0.8,
                pop=("uniform",), x=("gaussian", 1.0), alpha=0.5, T=3, seed=0,
                weighted=False, p_extra=10, name="custom", shuffle=True) -> ABG:
    """Draw one planted ABG. U nodes fall in k equal clusters, V in k equal blocks."""
    if m % k:
        raise ValueError("m must be a multiple of k (equal V blocks)")
    S = m // k
    rg = _rng(seed, "graph")
    rp = _rng(seed, "perm")
    cl = (np.arange(n, dtype=np.int64) * k) // n          # planted cluster by planted index
    degs = _draw_degrees(rg, n, deg)
    degs = np.minimum(degs, S)                               # cannot exceed one block's size
    u_pl = np.repeat(np.arange(n, dtype=np.int64), degs)
    v_pl = _draw_endpoints(rg, cl[u_pl], k, S, p_in, pop)
    u_pl, v_pl = _dedup_edges(rg, u_pl, v_pl, cl, k, S, m, p_in, pop)
    uperm = rp.permutation(n) if shuffle else np.arange(n)
    vperm = rp.permutation(m) if shuffle else np.arange(m)
    u_id = uperm[u_pl]
    v_id = vperm[v_pl]
    w = None
    if weighted:
        w = (_rng(seed, "aux").random(u_id.shape[0], dtype=np.float32) * 1.5 + 0.25).astype(np.float32)
    B_rowptr, B_col, Bt_rowptr, Bt_col, B_val, Bt_val = csr_from_edges(u_id, v_id, n, m, w)
    Xp = _draw_X(_rng(seed, "X"), n, d, k, cl, x)
    X = np.empty_like(Xp)
    X[uperm] = Xp
    truth = np.empty(n, np.int32)
    truth[uperm] = cl.astype(np.int32)
    G = _rng(seed, "G").standard_normal((d, d))
    Omega = _rng(seed, "Omega").standard_normal((2 * d, min(2 * d, k + p_extra))).astype(np.float32)
    return ABG(n=n, m=m, d=d, k=k, alpha=float(alpha), T=int(T), B_rowptr=B_rowptr, B_col=B_col,
               Bt_rowptr=Bt_rowptr, Bt_col=Bt_col, X=X, G=G, Omega=Omega, truth=truth,
               B_val=B_val, Bt_val=Bt_val, name=name, seed=seed)


def make_config(name: str, seed: int = 0, **over) -> ABG:
    """One of BASELINE.json's five configs (tiny, small, medium, large, xl)."""
    c = dict(CONFIGS[name])
    c.update(over)
    return planted_abg(c["n"], c["m"], c["k"], c["d"], deg=c["deg"], p_in=c["p_in"], pop=c["pop"],
                       x=c["x"], alpha=c["alpha"], T=c["T"], seed=seed, name=name)


def planted_rows(n: int, d: int, k: int, seed: int = 0, sigma: float = 1.0):
    """Planted Gaussian unit rows without a graph: k equal clusters in shuffled order, rows
    mu_c + sigma N(0, I) L2-normalised (the X recipe of the medium/large/xl configs), standing in
    for Zhat where a test needs the discretisation's launch shapes at a size whose graph would be
    too costly to propagate in the oracle.  Returns (rows fp32 [n, d], truth int32 [n])."""
    cl = (np.arange(n, dtype=np.int64) * k) // n
    Xp = _draw_X(_rng(seed, "X"), n, d, k, cl, ("gaussian", sigma))
    perm = _rng(seed, "perm").permutation(n)
    X = np.empty_like(Xp)
    X[perm] = Xp
    truth = np.empty(n, np.int32)
    truth[perm] = cl.astype(np.int32)
    return X, truth


def random_unit_rows(n: int, d: int, seed: int = 0, zero_rows=()) -> np.ndarray:
    """fp32 rows uniformly on the unit sphere (stage inputs standing in for Z-hat)."""
    r = _rng(seed, "aux").standard_normal((n, d)).astype(np.float32)
    r /= np.linalg.norm(r, axis=1, keepdims=True).astype(np.float32)
    for i in zero_rows:
        r[i] = 0
    return r
