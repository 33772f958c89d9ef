"""tpo_rowgemm_f64 (out = diag(rs) A W in fp64; Alg. 2's RH = dinv . (R' H), a7's Gamma) against an
fp64 reference: the integer-tensor-core path (Ozaki digit splitting, csrc/oz.cu) must stay within
its stated bound 2^-44 K max|A_i| max|W_l| |rs_i| of the exact product, and within a few units of
the fp64 DMMA path's own error."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tpo():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2405_11922_b200 import build
    build.build()
    import paper_2405_11922_b200 as T
    return T


def _ref(A, W, rs):
    out = A.astype(np.float64) @ W
    if rs is not None:
        out *= rs.astype(np.float64)[:, None]
    return out


def _bound(A, W, rs):
    K = A.shape[1]
    ma = np.abs(A.astype(np.float64)).max(axis=1)
    mw = np.abs(W).max(axis=0)
    r = np.abs(rs.astype(np.float64)) if rs is not None else np.ones(A.shape[0])
    return 2.0 ** -44 * K * np.outer(ma * r, mw) + 1e-300


def _case(rng, n, K, N, kind):
    if kind == "features":            # R'-like: amplitude * sin / cos values
        A = (np.sqrt(np.e / K) * np.sin(rng.uniform(-6, 6, (n, K)))).astype(np.float32)
        W = np.abs(rng.normal(size=(K, N))) * 0.1 + 1e-12
        W[rng.random((K, N)) < 0.2] = 1e-12              # R9 clamp floor entries
    elif kind == "signed":
        A = rng.normal(size=(n, K)).astype(np.float32)
        W = rng.normal(size=(K, N))
    else:                              # wide dynamic range inside rows and columns, zero rows
        A = (rng.normal(size=(n, K)) * 10.0 ** rng.uniform(-8, 3, (n, K))).astype(np.float32)
        A[::17] = 0.0
        W = rng.normal(size=(K, N)) * 10.0 ** rng.uniform(-10, 4, (K, N))
        W[:, 0] = 0.0
    rs = rng.uniform(0.2, 3.0, n).astype(np.float32)
    return A, W, rs


@pytest.mark.parametrize("n,K,N,kind", [(1000, 256, 50, "features"), (1000, 256, 50, "signed"),
                                        (777, 256, 64, "range"), (300, 100, 20, "signed"),
                                        (129, 64, 10, "features"), (5, 256, 16, "range"),
                                        (4000, 512, 20, "features"), (2000, 160, 33, "signed")])
def test_rowgemm_f64_bound(tpo, monkeypatch, n, K, N, kind):
    rng = np.random.default_rng(n + K + N)
    A, W, rs = _case(rng, n, K, N, kind)
    ref = _ref(A, W, rs)
    bound = _bound(A, W, rs)
    dA, dW, drs = torch.from_numpy(A).cuda(), torch.from_numpy(W).cuda(), torch.from_numpy(rs).cuda()
    out = tpo.rowgemm_f64(dA, dW, drs).cpu().numpy()
    err = np.abs(out - ref)
    assert np.all(err <= bound), (err / bound).max()
    out2 = tpo.rowgemm_f64(dA, dW, drs).cpu().numpy()
    assert np.array_equal(out, out2)                                    # deterministic
    monkeypatch.setenv("TPO_OZ", "0")
    dm = tpo.rowgemm_f64(dA, dW, drs).cpu().numpy()
    err_dm = np.abs(dm - ref)
    # the integer path is at least as close to the exact product as fp64 DMMA, up to 2^-44 K
    # max|A| max|W| (it truncates below that; DMMA rounds every partial sum)
    assert np.all(err <= err_dm + bound)
    out_n = tpo.rowgemm_f64(dA, dW, None).cpu().numpy()                 # rs = NULL
    monkeypatch.delenv("TPO_OZ")
    out_n2 = tpo.rowgemm_f64(dA, dW, None).cpu().numpy()
    ref_n = _ref(A, W, None)
    assert np.all(np.abs(out_n2 - ref_n) <= _bound(A, W, None))
    assert np.all(np.abs(out_n - ref_n) <= _bound(A, W, None))


def test_rowgemm_f64_many_tiles(tpo):
    """More row tiles than SMs (the persistent loop, ring and TMEM reuse across tiles), ragged
    last tile; large-config shape (K = 256, N = 50)."""
    rng = np.random.default_rng(7)
    n, K, N = 148 * 128 * 3 + 77, 256, 50
    A, W, rs = _case(rng, n, K, N, "features")
    out = tpo.rowgemm_f64(torch.from_numpy(A).cuda(), torch.from_numpy(W).cuda(), torch.from_numpy(rs).cuda())
    out = out.cpu().numpy()
    idx = rng.choice(n, 4000, replace=False)
    idx = np.concatenate([idx, np.arange(n - 200, n)])
    ref = _ref(A[idx], W, rs[idx])
    assert np.all(np.abs(out[idx] - ref) <= _bound(A[idx], W, rs[idx]))


# --------------------------------------------------------------------------------------------
# Alg. 2's R^T Ups = R'^T (dinv . Ups) on the integer tensor cores (oz_rtu_kernel, 32 < k <= 64)
# --------------------------------------------------------------------------------------------
def _rtu_case(rng, n, D, k, kind):
    A = (np.sqrt(np.e / (D // 2)) * np.sin(rng.uniform(-6, 6, (n, D)))).astype(np.float32)
    if kind == "cos":                                  # mostly positive columns: coherent sums
        A[:, D // 2:] = np.abs(A[:, D // 2:])
    U = np.abs(rng.normal(size=(n, k))) / np.sqrt(n) + 1e-12
    if kind == "range":
        U *= 10.0 ** rng.uniform(-9, 2, (n, k))
        U[:, 0] = 1e-12                               # R9 floor column
        A[::13] = 0.0
    dinv = rng.uniform(0.2, 3.0, n).astype(np.float32)
    return A, U, dinv


@pytest.mark.parametrize("n,D,k,kind", [(5000, 256, 50, "sin"), (70001, 260, 33, "cos"), (4099, 256, 49, "range"),
                                        (7, 256, 64, "sin"), (40000, 512, 64, "range"), (148 * 32 + 5, 128, 40, "cos")])
def test_onmf_rtu_integer_tensor_cores(tpo, monkeypatch, n, D, k, kind):
    """oz R^T Ups (B = dinv . Ups): within the kernel's rigorous bound of the exact sum, per row
    2^-52 2^EA 2^EB (dropped digit pairs, 2^E <= 2 max) + 2^-47 2^EA B_il + 2^-48 2^EB |R'_ij|
    (roundings); within 4e-14 of the L1 mass sum_i |R'_ij| B_il; close to the fp64 DMMA path;
    bitwise deterministic; ragged rows / feature tiles / odd k (the 8-byte Ups tail copy)."""
    rng = np.random.default_rng(n + D + k)
    A, U, dinv = _rtu_case(rng, n, D, k, kind)
    B = dinv.astype(np.float64)[:, None] * U
    ref = A.astype(np.float64).T @ B
    l1 = np.abs(A.astype(np.float64)).T @ B
    dA, dU, dd = torch.from_numpy(A).cuda(), torch.from_numpy(U).cuda(), torch.from_numpy(dinv).cuda()
    out = tpo.onmf_rtu(dA, dd, dU).cpu().numpy()
    err = np.abs(out - ref)
    mA, mB = 2 * np.abs(A).max(axis=0).astype(np.float64), 2 * B.max(axis=0)
    rig = (2.0 ** -52 * n * np.outer(mA, mB) + 2.0 ** -47 * np.outer(mA, B.sum(axis=0)) +
           2.0 ** -48 * np.outer(np.abs(A.astype(np.float64)).sum(axis=0), mB)) * 1.01 + 1e-300
    assert np.all(err <= rig), (err / rig).max()
    assert np.all(err <= 4e-14 * l1 + 1e-300), (err / (l1 + 1e-300)).max()
    assert np.array_equal(out, tpo.onmf_rtu(dA, dd, dU).cpu().numpy())     # deterministic
    monkeypatch.setenv("TPO_OZ", "0")
    dm = tpo.onmf_rtu(dA, dd, dU).cpu().numpy()
    monkeypatch.delenv("TPO_OZ")
    assert np.all(np.abs(dm - out) <= 4e-14 * l1 + 1e-300)
