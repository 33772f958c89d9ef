"""B200-native (sm_100a) implementation of the TPO hot path (arXiv 2405.11922).

The product is libtpo.so (C-ABI in include/tpo.h, CUDA sources in csrc/); this package is
its thin Python binding.  There is no CPU fallback: importing the binding functions needs
the built library (`python -m paper_2405_11922_b200.build`).
"""
from .tpo import (DeviceGraph, HostRunner, Runner, affinity_matvec, affinity_matvec_rfree, cluster, evaluate, features, gram, haar_q,  # noqa: F401
                  rowgemm_f64, onmf_rtu,
                  haar_q_dev, objective, propagate, run, svd_reduce, to_device_graph, topk_eig, topk_eig_rfree, cluster_rfree)
from ._lib import TPO_EIG_EXACT, TPO_EIG_HALKO, TpoError, lib  # noqa: F401
