"""Device-resident tprod time, int8 (Ozaki) vs DMMA stage 2, over shapes (decides the auto threshold)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2212_14318_b200 as qt
from paper_2212_14318_b200 import _native

L = _native.lib()
SHAPES = [(256, 256, 256, 64), (512, 512, 512, 64), (1024, 1024, 1024, 32), (256, 1024, 1024, 32),
          (1024, 1024, 256, 32), (1024, 256, 1024, 32), (1080, 1920, 64, 64), (1080, 1920, 128, 64),
          (2048, 2048, 2048, 8), (4096, 512, 512, 16)]


def run(m, n, s, p, algo, reps=5):
    dev = "cuda"
    mk = lambda r, c: torch.randn(2, p, r, c, dtype=torch.complex128, device=dev)
    ah, bh = mk(m, n), mk(n, s)
    c = torch.empty(2, p, m, s, dtype=torch.complex128, device=dev)
    f = lambda: _native.check(L.qt_spectral_product_f64_device_ld_algo(
        ah[0].data_ptr(), ah[1].data_ptr(), bh[0].data_ptr(), bh[1].data_ptr(), c[0].data_ptr(), c[1].data_ptr(),
        m, n, s, p, s, s, n * s, m * s, algo, None), "k2")
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for (m, n, s, p) in SHAPES:
    td = run(m, n, s, p, 0)
    t8 = run(m, n, s, p, 1)
    fl = 32 * m * n * s * p
    print(f"{(m, n, s, p)}: dmma {td:8.3f} ms ({fl / td / 1e9:6.1f} TF)  int8 {t8:8.3f} ms ({fl / t8 / 1e9:6.1f} TF)  "
          f"ratio {td / t8:5.2f}  auto={L.qt_gemm_algo(m, n, s, p)}", flush=True)
