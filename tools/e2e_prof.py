"""Per-kernel device time inside one e2e (host-buffer) T-product call (qt_prof_*)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2212_14318_b200 as qt
from paper_2212_14318_b200.configs import CONFIGS
cfg = CONFIGS[int(os.environ.get("CFG", 5))]
L = qt._native.lib()
a, b = qt.make_inputs(cfg)
pin = lambda x: torch.from_numpy(x.view('float64')).pin_memory()
a1, a2, b1, b2 = pin(a.t1), pin(a.t2), pin(b.t1), pin(b.t2)
c1 = torch.empty((cfg.p, cfg.m, 2 * cfg.s), dtype=torch.float64).pin_memory()
c2 = torch.empty_like(c1).pin_memory()
def run():
    qt._native.check(L.qt_tprod_f64_host(a1.data_ptr(), a2.data_ptr(), b1.data_ptr(), b2.data_ptr(), c1.data_ptr(),
                                         c2.data_ptr(), cfg.m, cfg.n, cfg.s, cfg.p, 0), "host")
run()
t0 = time.perf_counter(); run(); print("e2e ms", (time.perf_counter() - t0) * 1e3)
L.qt_prof_enable(1); run(); L.qt_prof_enable(0)
for tag in ("fft", "k2_dmma", "k2_dmma_guard", "k2_int8_gemm", "k2_int8_residues", "k2_int8_crt"):
    ms, n = ctypes.c_double(), ctypes.c_uint64()
    L.qt_prof_read(tag.encode(), ctypes.byref(ms), ctypes.byref(n))
    if n.value: print(f"{tag:18s} {ms.value:8.2f} ms  {n.value} launches")
