#!/bin/bash
# Build the CSR gather probe and run it on the small config's two SpMM index streams.
set -e
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gather_csr tools/probes/gather_csr.cu
python - <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np
from synth import make_config
g = make_config("small")
g.Bt_col.astype(np.int32).tofile('/tmp/bt_col.bin')   # SpMM-1 gathers P rows (n) by Bt col ids
g.B_col.astype(np.int32).tofile('/tmp/b_col.bin')     # SpMM-2 gathers Q rows (m) by B col ids
print(g.n, g.m, g.d)
PY
/tmp/gather_csr /tmp/bt_col.bin 50000 1000
/tmp/gather_csr /tmp/b_col.bin 80000 1000
