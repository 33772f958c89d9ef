"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This package holds NO arithmetic of the TPO method (no degree normalisation, no
propagation, no features): it only draws planted-cluster attributed bipartite graphs
(ABGs) and the random matrices the method consumes (G for the Haar rotation of
Alg. 1 L6; Omega for the randomised SVD of Alg. 2 L1).
The recipes are the SURVEY.md §8(d) readings of BASELINE.json's configs; DESIGN.md
restates them.
"""
from .generate import CONFIGS, ABG, make_config, planted_abg, planted_rows, csr_from_edges, random_unit_rows  # noqa: F401
