"""Bitwise check of the int8 stage 2 between two runs: the first saves its
outputs, later runs compare against them — e.g. QTB_OZAKI_SHAREX=0 vs 1 (shared
X' within a pair), or QTB_CHECK_LIB=<another build of the library> vs this one."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2212_14318_b200 import _native
if os.environ.get("QTB_CHECK_LIB"):  # compare another build of the library (e.g. the previous commit's)
    import ctypes
    L = ctypes.CDLL(os.environ["QTB_CHECK_LIB"])
    for name, (res, args) in _native.SIGNATURES.items():
        if hasattr(L, name):
            getattr(L, name).restype, getattr(L, name).argtypes = res, args
else:
    L = _native.lib()
out = sys.argv[1]
res = {}
for (m, n, s, p) in [(150, 256, 520, 6), (64, 256, 256, 5), (300, 512, 384, 8), (33, 256, 130, 2), (2048, 2048, 2048, 4)]:
    g = torch.Generator(device="cuda").manual_seed(m + n + s + p)
    ah = torch.randn((2, p, m, 2 * n), dtype=torch.float64, device="cuda", generator=g)
    bh = torch.randn((2, p, n, 2 * s), dtype=torch.float64, device="cuda", generator=g)
    ch = torch.zeros((2, p, m, 2 * s), dtype=torch.float64, device="cuda")
    _native.check(L.qt_spectral_product_f64_device_ld_algo(ah[0].data_ptr(), ah[1].data_ptr(), bh[0].data_ptr(),
                                                           bh[1].data_ptr(), ch[0].data_ptr(), ch[1].data_ptr(),
                                                           m, n, s, p, s, s, n * s, m * s, 1, None), "int8")
    res[f"{m}_{n}_{s}_{p}"] = ch.cpu().numpy()
if os.path.exists(out):
    ref = np.load(out)
    for k, v in res.items():
        same = np.array_equal(ref[k].view(np.uint64), v.view(np.uint64))
        print(k, "bitwise equal" if same else f"DIFFERENT max {np.abs(ref[k] - v).max()}")
else:
    np.savez(out, **res)
    print("saved", list(res))
