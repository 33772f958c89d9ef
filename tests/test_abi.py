"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, exports every symbol
include/tpo.h declares, validates arguments before touching the GPU, and its host-only
entry point (tpo_haar_q) agrees with the oracle's independent QR."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2405_11922_b200 import build
    build.build()
    from paper_2405_11922_b200 import _lib
    return _lib.lib()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "tpo.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tpo_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    from paper_2405_11922_b200 import _lib
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(L, s), f"libtpo.so does not export {s}"
    assert set(syms) == set(_lib.SYMBOLS)
    assert L.tpo_abi_version() == 1


def test_sm100a_cubin(L):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", os.path.join(ROOT, "paper_2405_11922_b200", "libtpo.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_validation_errors_without_gpu(L):
    from paper_2405_11922_b200._lib import CSR, TPO_EINVAL, TPO_ENOMEM
    B = CSR(10, 5, 0, 16, 0, None)
    Bt = CSR(5, 10, 0, 16, 0, None)
    rc = L.tpo_propagate(C.byref(B), C.byref(Bt), None, 8, 0.5, 2, None, None, None, 0, None)
    assert rc == TPO_EINVAL and b"X is NULL" in L.tpo_last_error()
    rc = L.tpo_propagate(C.byref(B), C.byref(Bt), 16, 8, 1.5, 2, 16, None, None, 0, None)
    assert rc == TPO_EINVAL and b"alpha" in L.tpo_last_error()
    rc = L.tpo_propagate(C.byref(B), C.byref(Bt), 16, 6, 0.5, 2, 16, None, None, 0, None)
    assert rc == TPO_EINVAL and b"multiple of 4" in L.tpo_last_error()
    Bt_bad = CSR(5, 10, 3, 16, 16, None)
    rc = L.tpo_propagate(C.byref(B), C.byref(Bt_bad), 16, 8, 0.5, 2, 16, None, None, 0, None)
    assert rc == TPO_EINVAL and b"nnz" in L.tpo_last_error()
    rc = L.tpo_propagate(C.byref(B), C.byref(Bt), 16, 8, 0.5, 2, 16, None, 256, 10, None)
    assert rc == TPO_ENOMEM
    # gathered tables of >= 2^32 float4 would wrap the SpMM's 32-bit gather offsets: rejected
    # (20 M U rows at d = 1000 is 5e9 float4)
    Bbig = CSR(20_000_000, 5, 0, 16, 0, None)
    Btbig = CSR(5, 20_000_000, 0, 16, 0, None)
    rc = L.tpo_propagate(C.byref(Bbig), C.byref(Btbig), 16, 1000, 0.5, 2, 16, None, None, 0, None)
    assert rc == TPO_EINVAL and b"32-bit gather offsets" in L.tpo_last_error()
    Bwide = CSR(5, 20_000_000, 0, 16, 0, None)       # V side too large (gathered by the U-side SpMM)
    Btwide = CSR(20_000_000, 5, 0, 16, 0, None)
    rc = L.tpo_propagate(C.byref(Bwide), C.byref(Btwide), 16, 1000, 0.5, 2, 16, None, None, 0, None)
    assert rc == TPO_EINVAL and b"32-bit gather offsets" in L.tpo_last_error()
    rc = L.tpo_shard_vside(C.byref(Btbig), 16, 1000, 16, None, 0, None)
    assert rc == TPO_EINVAL and b"32-bit gather offsets" in L.tpo_last_error()
    rc = L.tpo_shard_uside(C.byref(Bwide), 16, 16, 1000, 0.5, 16, 0, 16, None, None, 0, None)
    assert rc == TPO_EINVAL and b"32-bit gather offsets" in L.tpo_last_error()
    rc = L.tpo_topk_eig(16, 16, 100, 8, 9, 0, 0, 0, None, 16, None, 16, 256, 1 << 30, None)
    assert rc == TPO_EINVAL and b"k must" in L.tpo_last_error()
    h = C.c_void_p()
    rc = L.tpo_comm_create(C.create_string_buffer(128), 2, 2, 0, C.byref(h))   # rank >= world
    assert rc == TPO_EINVAL and b"rank" in L.tpo_last_error()
    rc = L.tpo_svd_reduce(16, 100, 64, 65, 16, None, 256, 1 << 30, None)       # d > d_u
    assert rc == TPO_EINVAL and b"d must" in L.tpo_last_error()
    rc = L.tpo_svd_reduce(16, 100, 62, 8, 16, None, 256, 1 << 30, None)        # d_u % 4
    assert rc == TPO_EINVAL and b"d_u" in L.tpo_last_error()
    rc = L.tpo_topk_eig(16, 16, 100, 8, 2, 7, 0, 0, None, 16, None, 16, 256, 1 << 30, None)
    assert rc == TPO_EINVAL and b"mode" in L.tpo_last_error()


def test_workspace_queries(L):
    assert L.tpo_propagate_ws(2_000_000, 1_000_000, 60_000_000, 128) > 1_000_000 * 128 * 4
    assert L.tpo_features_ws(1000, 300) > 0
    assert L.tpo_topk_eig_ws(1000, 600, 5, 0, 10) > 600 * 600 * 8
    assert L.tpo_cluster_ws(1000, 600, 5) > 1000 * 5 * 8
    assert L.tpo_run_ws(2000, 3000, 16000, 300, 5, 0, 10) > 0


@pytest.mark.parametrize("d", [1, 3, 17, 64])
def test_haar_q_matches_oracle(L, d):
    """tpo_haar_q (library: Gram-Schmidt with re-orthogonalisation) vs the oracle's Householder
    QR: the positive-diagonal QR is unique, so both must return the same Q."""
    from oracle import core as O
    from paper_2405_11922_b200 import haar_q
    G = np.random.default_rng(d).standard_normal((d, d))
    Q = haar_q(G)
    assert np.allclose(Q, O.haar_q(G), atol=1e-12)
