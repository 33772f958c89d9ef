"""ctypes loader of the in-tree libtpo.so (the C-ABI of include/tpo.h).

Loading fails loudly: there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtpo.so")

# exported symbols, as declared in include/tpo.h
SYMBOLS = [
    "tpo_abi_version", "tpo_last_error", "tpo_launch_count",
    "tpo_propagate_ws", "tpo_propagate",
    "tpo_shard_ws", "tpo_shard_degrees", "tpo_shard_start", "tpo_shard_vside", "tpo_shard_vscale", "tpo_shard_uside", "tpo_haar_q", "tpo_haar_q_dev_ws", "tpo_haar_q_dev",
    "tpo_features_ws", "tpo_features",
    "tpo_affinity_matvec_ws", "tpo_affinity_matvec",
    "tpo_gram_ws", "tpo_gram", "tpo_topk_eig_ws", "tpo_topk_eig",
    "tpo_cluster_ws", "tpo_cluster",
    "tpo_run_ws", "tpo_run", "tpo_run_host_ws", "tpo_run_host",
    "tpo_shard_solver_ws", "tpo_shard_features", "tpo_shard_dinv", "tpo_eig_from_gram", "tpo_shard_gamma",
    "tpo_shard_atb64", "tpo_shard_apply_chol", "tpo_shard_colstats", "tpo_shard_gamma_final",
    "tpo_shard_onmf_init", "tpo_shard_onmf_rtu", "tpo_onmf_h_update", "tpo_shard_onmf_rh",
    "tpo_rowgemm_f64_ws", "tpo_rowgemm_f64",
    "tpo_shard_onmf_u_update", "tpo_shard_nci_assign", "tpo_nci_phi",
    "tpo_svd_reduce_ws", "tpo_svd_reduce", "tpo_eval_ws", "tpo_eval", "tpo_objective_ws", "tpo_objective",
    "tpo_rows_gather", "tpo_rows_scatter",
    "tpo_comm_unique_id", "tpo_comm_create", "tpo_comm_destroy", "tpo_propagate_sharded_ws", "tpo_propagate_sharded",
    "tpo_affinity_matvec_rfree_ws", "tpo_affinity_matvec_rfree", "tpo_run_sharded_ws", "tpo_run_sharded",
    "tpo_topk_eig_rfree_ws", "tpo_topk_eig_rfree", "tpo_cluster_rfree_ws", "tpo_cluster_rfree",
]

TPO_OK, TPO_EINVAL, TPO_ECUDA, TPO_ENOMEM, TPO_ENCCL, TPO_ENUMERIC = 0, -1, -2, -3, -4, -5
TPO_EIG_EXACT, TPO_EIG_HALKO = 0, 1
_NAMES = {-1: "TPO_EINVAL", -2: "TPO_ECUDA", -3: "TPO_ENOMEM", -4: "TPO_ENCCL", -5: "TPO_ENUMERIC"}


class TpoError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_NAMES.get(code, code)}: {msg}")
        self.code = code


class CSR(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_cols", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("val", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libtpo.so not built at {LIB_PATH}: run `python -m paper_2405_11922_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    i64, i32, sz, vp, f32, dbl = C.c_int64, C.c_int32, C.c_size_t, C.c_void_p, C.c_float, C.c_double
    P = C.POINTER(CSR)
    L.tpo_abi_version.restype = C.c_int
    L.tpo_last_error.restype = C.c_char_p
    L.tpo_launch_count.restype = C.c_uint64
    L.tpo_propagate_ws.argtypes = [i64, i64, i64, i64]
    L.tpo_propagate_ws.restype = sz
    L.tpo_propagate.argtypes = [P, P, vp, i64, f32, i32, vp, vp, vp, sz, vp]
    L.tpo_shard_ws.argtypes = [i64, i64, i64]
    L.tpo_shard_ws.restype = sz
    L.tpo_shard_degrees.argtypes = [P, P, vp, vp, vp]
    L.tpo_shard_start.argtypes = [vp, vp, i64, i64, vp, i64, f32, vp, vp, vp, vp]
    L.tpo_shard_vside.argtypes = [P, vp, i64, vp, vp, sz, vp]
    L.tpo_shard_vscale.argtypes = [vp, vp, i64, i64, vp]
    L.tpo_shard_uside.argtypes = [P, vp, vp, i64, f32, vp, i32, vp, vp, vp, sz, vp]
    L.tpo_haar_q.argtypes = [vp, i64, vp]
    L.tpo_haar_q_dev_ws.argtypes = [i64]
    L.tpo_haar_q_dev_ws.restype = sz
    L.tpo_haar_q_dev.argtypes = [vp, i64, vp, vp, sz, vp]
    L.tpo_features_ws.argtypes = [i64, i64]
    L.tpo_features_ws.restype = sz
    L.tpo_features.argtypes = [vp, i64, i64, vp, vp, vp, vp, vp, sz, vp]
    L.tpo_affinity_matvec_ws.argtypes = [i64, i64, i64]
    L.tpo_affinity_matvec_ws.restype = sz
    L.tpo_affinity_matvec.argtypes = [vp, vp, i64, i64, vp, i64, vp, vp, sz, vp]
    L.tpo_gram_ws.argtypes = [i64, i64]
    L.tpo_gram_ws.restype = sz
    L.tpo_gram.argtypes = [vp, vp, i64, i64, vp, vp, sz, vp]
    L.tpo_topk_eig_ws.argtypes = [i64, i64, i32, i32, i32]
    L.tpo_topk_eig_ws.restype = sz
    L.tpo_topk_eig.argtypes = [vp, vp, i64, i64, i32, i32, i32, i32, vp, vp, vp, vp, vp, sz, vp]
    L.tpo_cluster_ws.argtypes = [i64, i64, i32]
    L.tpo_cluster_ws.restype = sz
    L.tpo_cluster.argtypes = [vp, vp, i64, i64, i32, vp, vp, vp, i32, i32, vp, vp, vp, sz, vp]
    L.tpo_run_ws.argtypes = [i64, i64, i64, i64, i32, i32, i32]
    L.tpo_run_ws.restype = sz
    L.tpo_run.argtypes = [P, P, vp, i64, f32, i32, i32, vp, i32, vp, i32, i32, i32, i32, vp, vp, vp, sz, vp]
    L.tpo_run_host_ws.argtypes = [i64, i64, i64, i64, i32, i32, i32, i32]
    L.tpo_run_host_ws.restype = sz
    L.tpo_run_host.argtypes = [P, P, vp, i64, f32, i32, i32, vp, i32, vp, i32, i32, i32, i32, vp, vp, vp, sz, vp]
    L.tpo_shard_solver_ws.argtypes = [i64, i64, i32]
    L.tpo_shard_solver_ws.restype = sz
    L.tpo_shard_features.argtypes = [vp, i64, i64, vp, vp, vp, vp, sz, vp]
    L.tpo_shard_dinv.argtypes = [vp, i64, i64, vp, vp, vp]
    L.tpo_eig_from_gram.argtypes = [vp, vp, i64, i32, vp, vp, vp, sz, vp]
    L.tpo_shard_gamma.argtypes = [vp, vp, i64, i64, i32, vp, vp, vp, vp, sz, vp]
    L.tpo_shard_atb64.argtypes = [vp, vp, i64, i32, vp, vp, sz, vp]
    L.tpo_shard_apply_chol.argtypes = [vp, i64, i32, vp, vp, sz, vp]
    L.tpo_shard_colstats.argtypes = [vp, i64, i32, i64, vp, vp, vp, vp, vp, sz, vp]
    L.tpo_shard_gamma_final.argtypes = [vp, i64, i32, vp, vp, i64, vp, vp, vp, sz, vp]
    L.tpo_shard_onmf_init.argtypes = [vp, i64, vp, vp, i64, i32, vp, vp, vp, sz, vp]
    L.tpo_shard_onmf_rtu.argtypes = [vp, vp, vp, i64, i64, i32, vp, vp, sz, vp]
    L.tpo_onmf_h_update.argtypes = [vp, vp, vp, i64, i32, vp, sz, vp]
    L.tpo_shard_onmf_rh.argtypes = [vp, vp, vp, i64, i64, i32, vp, vp]
    L.tpo_shard_onmf_u_update.argtypes = [vp, vp, vp, i64, i32, vp]
    L.tpo_shard_nci_assign.argtypes = [vp, vp, i64, i32, vp, vp, vp, vp, vp, sz, vp]
    L.tpo_nci_phi.argtypes = [vp, vp, i32, vp, vp]
    L.tpo_svd_reduce_ws.argtypes = [i64, i64, i64]
    L.tpo_svd_reduce_ws.restype = sz
    L.tpo_svd_reduce.argtypes = [vp, i64, i64, i64, vp, vp, vp, sz, vp]
    L.tpo_svd_reduce.restype = C.c_int
    L.tpo_eval_ws.argtypes = [i32, i32]
    L.tpo_eval_ws.restype = sz
    L.tpo_eval.argtypes = [vp, vp, i64, i32, i32, vp, vp, sz, vp]
    L.tpo_eval.restype = C.c_int
    L.tpo_objective_ws.argtypes = [i64, i64, i32]
    L.tpo_objective_ws.restype = sz
    L.tpo_objective.argtypes = [vp, vp, i64, i64, i32, vp, vp, vp, vp, sz, vp]
    L.tpo_objective.restype = C.c_int
    L.tpo_rows_gather.argtypes = [vp, vp, i64, i64, vp, vp]
    L.tpo_rows_gather.restype = C.c_int
    L.tpo_rows_scatter.argtypes = [vp, vp, i64, i64, vp, i32, vp]
    L.tpo_rows_scatter.restype = C.c_int
    L.tpo_comm_unique_id.argtypes = [vp]
    L.tpo_comm_unique_id.restype = C.c_int
    L.tpo_comm_create.argtypes = [vp, i32, i32, i32, C.POINTER(C.c_void_p)]
    L.tpo_comm_create.restype = C.c_int
    L.tpo_comm_destroy.argtypes = [vp]
    L.tpo_comm_destroy.restype = C.c_int
    L.tpo_propagate_sharded_ws.argtypes = [i64, i64, i64, i64, i32]
    L.tpo_propagate_sharded_ws.restype = sz
    L.tpo_propagate_sharded.argtypes = [vp, P, P, vp, i64, f32, i32, vp, vp, vp, sz, vp]
    L.tpo_propagate_sharded.restype = C.c_int
    L.tpo_affinity_matvec_rfree_ws.argtypes = [i64, i64, i64, i64]
    L.tpo_affinity_matvec_rfree_ws.restype = sz
    L.tpo_affinity_matvec_rfree.argtypes = [vp, i64, i64, vp, vp, i64, vp, i64, vp, sz, vp]
    L.tpo_affinity_matvec_rfree.restype = C.c_int
    L.tpo_topk_eig_rfree_ws.argtypes = [i64, i64, i32, i64]
    L.tpo_topk_eig_rfree_ws.restype = sz
    L.tpo_topk_eig_rfree.argtypes = [vp, i64, i64, vp, i32, vp, vp, vp, vp, i64, vp, sz, vp]
    L.tpo_topk_eig_rfree.restype = C.c_int
    L.tpo_cluster_rfree_ws.argtypes = [i64, i64, i32, i64]
    L.tpo_cluster_rfree_ws.restype = sz
    L.tpo_cluster_rfree.argtypes = [vp, i64, i64, vp, vp, i32, vp, vp, vp, i32, i32, vp, vp, i64, vp, sz, vp]
    L.tpo_cluster_rfree.restype = C.c_int
    L.tpo_rowgemm_f64_ws.argtypes = [i64, i64, i32]
    L.tpo_rowgemm_f64_ws.restype = sz
    L.tpo_rowgemm_f64.argtypes = [vp, i64, i64, vp, vp, i32, vp, vp, sz, vp]
    L.tpo_rowgemm_f64.restype = C.c_int
    L.tpo_run_sharded_ws.argtypes = [i64, i64, i64, i64, i32, i32]
    L.tpo_run_sharded_ws.restype = sz
    L.tpo_run_sharded.argtypes = [vp, P, P, vp, i64, f32, i32, i32, vp, i64, i32, i32, vp, vp, vp, vp, sz, vp]
    L.tpo_run_sharded.restype = C.c_int
    for name in ["tpo_shard_features", "tpo_shard_dinv", "tpo_eig_from_gram", "tpo_shard_gamma", "tpo_shard_atb64",
                 "tpo_shard_apply_chol", "tpo_shard_colstats", "tpo_shard_gamma_final", "tpo_shard_onmf_init",
                 "tpo_shard_onmf_rtu", "tpo_onmf_h_update", "tpo_shard_onmf_rh", "tpo_shard_onmf_u_update",
                 "tpo_shard_nci_assign", "tpo_nci_phi"]:
        getattr(L, name).restype = C.c_int
    for name in ["tpo_propagate", "tpo_shard_degrees", "tpo_shard_start", "tpo_shard_vside", "tpo_shard_vscale",
                 "tpo_shard_uside", "tpo_haar_q", "tpo_haar_q_dev", "tpo_features", "tpo_affinity_matvec", "tpo_gram", "tpo_topk_eig",
                 "tpo_cluster", "tpo_run", "tpo_run_host"]:
        getattr(L, name).restype = C.c_int
    _lib = L
    return L


def check(rc: int):
    if rc != TPO_OK:
        raise TpoError(rc, lib().tpo_last_error().decode())
