#!/usr/bin/env python3
"""Badly scaled contraction indices through the int8 stage 2 (accuracy guard
+ balancing, csrc/qt_ozaki.cu), checked against the reference restatement.

Prints one JSON line {case: {"err": rel. Frobenius error of tprod_fast vs
oracle.tprod_fast, "fallbacks": pairs sent to the fp64 DMMA kernels}} plus
"forced_bitwise_dmma": whether stage 2 with every pair forced to the fallback
equals the DMMA path bitwise.  Run under different $QTB_OZAKI_BALANCE /
$QTB_OZAKI_GUARD settings by tests/test_gpu_int8.py (the switches are read
once per process).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_2212_14318_b200 as qt  # noqa: E402
from paper_2212_14318_b200 import _native  # noqa: E402


def scaled_inputs(case, m, n, s, p, seed=5):
    a = qt.gen_random_tensor(m, n, p, seed)
    b = qt.gen_random_tensor(n, s, p, seed + 1)
    rng = np.random.default_rng(seed)
    a1, a2, b1, b2 = a.t1.copy(), a.t2.copy(), b.t1.copy(), b.t2.copy()
    if case.startswith("col"):  # one contraction index: A column x d, B row / d
        d, k = float(case[3:]), 7
        for t in (a1, a2):
            t[:, :, k] *= d
        for t in (b1, b2):
            t[:, k, :] /= d
    elif case == "logu_pair":  # every contraction index 2^U(-30, 30), inverse in B
        d = np.ldexp(1.0, rng.integers(-30, 31, n))
        for t in (a1, a2):
            t *= d[None, None, :]
        for t in (b1, b2):
            t /= d[None, :, None]
    elif case == "logu_a":  # A's columns only
        d = np.ldexp(1.0, rng.integers(-30, 31, n))
        for t in (a1, a2):
            t *= d[None, None, :]
    elif case == "logu_b_rows":  # B's rows only
        d = np.ldexp(1.0, rng.integers(-30, 31, n))
        for t in (b1, b2):
            t *= d[None, :, None]
    elif case == "one_elem":  # one huge entry of A
        a1[3, 5, 9] *= 1e8
    elif case != "plain":
        raise ValueError(case)
    return qt.CdTensor3(m, n, p, a1, a2), qt.CdTensor3(n, s, p, b1, b2)


def main():
    m, n, s, p = 64, 512, 256, 8
    L = _native.lib()
    assert L.qt_gemm_algo(m, n, s, p) == 1
    out = {}
    for case in ("plain", "col1e4", "col1e8", "logu_pair", "logu_a", "logu_b_rows", "one_elem"):
        a, b = scaled_inputs(case, m, n, s, p)
        f0 = L.qt_int8_guard_fallbacks()
        c = qt.tprod_fast(a, b)
        fb = L.qt_int8_guard_fallbacks() - f0
        err = O.rel_frob_error((c.t1, c.t2), O.tprod_fast((a.t1, a.t2), (b.t1, b.t2)))
        out[case] = {"err": err, "fallbacks": int(fb)}
    # stage 2 alone: int8 call vs DMMA call on the same operands
    import torch
    g = torch.Generator(device="cuda").manual_seed(3)
    ah = torch.randn((2, p, m, n), dtype=torch.complex128, device="cuda", generator=g)
    bh = torch.randn((2, p, n, s), dtype=torch.complex128, device="cuda", generator=g)
    res = []
    for algo in (1, 0):
        cc = torch.zeros((2, p, m, s), dtype=torch.complex128, device="cuda")
        _native.check(L.qt_spectral_product_f64_device_ld_algo(
            ah[0].data_ptr(), ah[1].data_ptr(), bh[0].data_ptr(), bh[1].data_ptr(), cc[0].data_ptr(),
            cc[1].data_ptr(), m, n, s, p, s, s, n * s, m * s, algo, None), "spectral")
        torch.cuda.synchronize()
        res.append(cc.cpu().numpy())
    out["forced_bitwise_dmma"] = bool(np.array_equal(res[0].view(np.uint64), res[1].view(np.uint64)))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
