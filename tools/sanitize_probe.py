#!/usr/bin/env python3
"""Small end-to-end exercise of every kernel family for compute-sanitizer runs
(one tool per gpurun call): tube FFT (single pass, fft2, four-step split,
global multi-pass), both GEMM tile shapes + the persistent small kernel,
the definitional product, QT3 I/O, the tiled host path and the multi driver."""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2212_14318_b200 as qt  # noqa: E402
from paper_2212_14318_b200 import tensor_io  # noqa: E402

for (m, n, s, p) in [(5, 4, 3, 6), (33, 17, 40, 16), (70, 64, 20, 64), (16, 16, 16, 4096), (2, 3, 2, 97),
                     (1, 2, 1, 8192), (130, 40, 150, 32), (3, 20, 5, 7)]:
    a = qt.gen_random_tensor(m, n, p, 1)
    b = qt.gen_random_tensor(n, s, p, 2)
    c = qt.tprod_fast(a, b)
    assert np.isfinite(c.t1).all()
    if p <= 64:
        qt.tprod_naive(a, b)
    qt.qifft3_conj(qt.qfft3_conj(a))
a = qt.gen_random_tensor(300, 64, 32, 3)
b = qt.gen_random_tensor(64, 200, 32, 4)
qt.tprod_fast(a, b)                 # tiled host path (>= 128 MB? no: exercise multi instead)
qt.tprod_fast_multi(a, b, [0])      # NCCL pipeline at G = 1
with tempfile.TemporaryDirectory() as d:
    tensor_io.write_tensor(os.path.join(d, "t.qt3"), a)
    tensor_io.read_tensor(os.path.join(d, "t.qt3"))
print("sanitize probe ok")
