#!/usr/bin/env python3
"""Small end-to-end exercise of every kernel family for compute-sanitizer runs
(memcheck / racecheck / synccheck): tube FFT (single pass, fft2, four-step
split, global multi-pass), both GEMM tile shapes + the persistent small
kernel, the int8 stage 2 (balancing, residues, tcgen05 CTA-pair GEMM, CRT,
accuracy guard, the per-pair fp64 fallback and the non-finite fallback), the
definitional product, QT3 I/O and the multi driver."""
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
# int8 stage 2 (auto-selected shapes), a pair the guard rejects, a non-finite input
for (m, n, s, p) in [(6, 256, 512, 4), (40, 256, 520, 5)]:
    a = qt.gen_random_tensor(m, n, p, 5)
    b = qt.gen_random_tensor(n, s, p, 6)
    assert qt._native.lib().qt_gemm_algo(m, n, s, p) == 1
    c = qt.tprod_fast(a, b)
    assert np.isfinite(c.t1).all()
a.t1[1, 3, 7] *= 1e12  # one huge entry: the guard sends its pair to the fp64 kernels
qt.tprod_fast(a, b)
a.t2[0, 2, 5] = float("inf")
qt.tprod_fast(a, b)
a = qt.gen_random_tensor(300, 64, 32, 3)
b = qt.gen_random_tensor(64, 200, 32, 4)
qt.tprod_fast(a, b)                 # tiled host path (>= 128 MB? no: exercise multi instead)
qt.tprod_fast_multi(a, b, [0])      # NCCL pipeline at G = 1
with tempfile.TemporaryDirectory() as d:
    tensor_io.write_tensor(os.path.join(d, "t.qt3"), a)
    tensor_io.read_tensor(os.path.join(d, "t.qt3"))
print("sanitize probe ok")
