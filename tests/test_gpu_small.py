"""The one-launch small-product kernel (csrc/qt_small.cu): a cluster of p/2 CTAs
per 8 x 16 block of C runs K1, K2 and K3 exchanging through distributed
shared memory.  It must give BITWISE the three-launch result (same
butterflies, twiddles and DMMA sequence), which the tests check against a
subprocess with the kernel switched off ($QTB_SMALL=0), plus the reference
restated (oracle, <= 1e-12) and the definitional product.  The product it
replaces is tprod_fast (/root/reference/proj/src/tproduct.cpp:75-111)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
import paper_2212_14318_b200 as qt
from paper_2212_14318_b200 import _native

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# config 1; edges of the 8 x 16 cluster block (rows, columns, K padding to 16,
# n = 1, the largest n) for every supported p
SHAPES = [(32, 32, 32, 16), (8, 8, 8, 4), (24, 20, 17, 8), (5, 64, 31, 16), (32, 1, 32, 4), (1, 16, 1, 16),
          (9, 48, 3, 8), (17, 7, 16, 16), (31, 33, 29, 4), (13, 20, 30, 2)]


def bits(x):
    return np.ascontiguousarray(x).view(np.uint64)


def inputs(m, n, s, p, k):
    a = O.gen_random_tensor(m, n, p, 900 + 2 * k)
    b = O.gen_random_tensor(n, s, p, 901 + 2 * k)
    if k == 2:  # non-finite values propagate the same way on both paths
        a[0][1, 0, 2] = np.inf
        b[1][0, 1, 0] = complex(np.nan, 1.0)
    return a, b


_THREE_LAUNCH = """
import json, sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import oracle as O, paper_2212_14318_b200 as qt
from test_gpu_small import SHAPES, inputs
L = qt._native.lib()
out = {{}}
for k, (m, n, s, p) in enumerate(SHAPES):
    assert L.qt_small_fused(m, n, s, p) == 0
    a, b = inputs(m, n, s, p, k)
    c = qt.tprod_fast(qt.CdTensor3(m, n, p, a[0], a[1]), qt.CdTensor3(n, s, p, b[0], b[1]))
    np.save({path!r} + f"_{{k}}_1.npy", c.t1); np.save({path!r} + f"_{{k}}_2.npy", c.t2)
print("ok")
"""


@pytest.fixture(scope="module")
def three_launch(tmp_path_factory):
    path = str(tmp_path_factory.mktemp("small") / "c")
    env = dict(os.environ, QTB_SMALL="0")
    code = _THREE_LAUNCH.format(root=ROOT, tests=os.path.join(ROOT, "tests"), path=path)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]
    return path


def test_selection():
    L = _native.lib()
    assert L.qt_small_fused(32, 32, 32, 16) == 1  # config 1
    assert L.qt_small_fused(32, 64, 32, 8) == 1
    assert L.qt_small_fused(33, 32, 32, 16) == 0  # beyond the small DMMA tiles
    assert L.qt_small_fused(32, 65, 32, 16) == 0  # operands exceed shared memory
    assert L.qt_small_fused(32, 32, 32, 12) == 0  # p not in {2, 4, 8, 16}
    assert L.qt_small_fused(32, 32, 32, 2) == 1
    assert L.qt_small_fused(16, 16, 16, 4096) == 0  # config 3


@pytest.mark.parametrize("k", range(len(SHAPES)))
def test_bitwise_three_launch_and_parity(three_launch, k):
    m, n, s, p = SHAPES[k]
    L = _native.lib()
    assert L.qt_small_fused(m, n, s, p) == 1
    a, b = inputs(m, n, s, p, k)
    before = L.qt_kernel_launches()
    c = qt.tprod_fast(qt.CdTensor3(m, n, p, a[0], a[1]), qt.CdTensor3(n, s, p, b[0], b[1]))
    assert L.qt_kernel_launches() - before == 1
    w1 = np.load(three_launch + f"_{k}_1.npy")
    w2 = np.load(three_launch + f"_{k}_2.npy")
    assert np.array_equal(bits(c.t1), bits(w1)) and np.array_equal(bits(c.t2), bits(w2)), (m, n, s, p)
    if k != 2:
        got = (c.t1, c.t2)
        assert O.rel_frob_error(got, O.tprod_fast(a, b)) <= 1e-12
        assert O.rel_frob_error(got, O.tprod_naive(a, b)) <= 1e-11


def test_device_entry_replay_and_row_slabs():
    """Through qt_tprod_f64_device (graph-recorded after the first call): one
    launch per call, bitwise equal to the host entry; row slabs of it (each
    its own one-launch product) stitch to the full product bitwise."""
    import torch
    L = _native.lib()
    m, n, s, p = 32, 32, 32, 16
    dev = torch.device("cuda", 0)
    a = qt.gen_random_tensor(m, n, p, 41)
    b = qt.gen_random_tensor(n, s, p, 42)
    want = qt.tprod_fast(a, b)
    da = [torch.from_numpy(x.view(np.float64)).to(dev) for x in (a.t1, a.t2)]
    db = [torch.from_numpy(x.view(np.float64)).to(dev) for x in (b.t1, b.t2)]
    dc = [torch.empty((p, m, 2 * s), dtype=torch.float64, device=dev) for _ in range(2)]
    for i in range(3):
        before = L.qt_kernel_launches()
        _native.check(L.qt_tprod_f64_device(da[0].data_ptr(), da[1].data_ptr(), db[0].data_ptr(), db[1].data_ptr(),
                                            dc[0].data_ptr(), dc[1].data_ptr(), m, n, s, p, None), "tprod")
        torch.cuda.synchronize()
        assert L.qt_kernel_launches() - before == 1
        got = [x.cpu().numpy().view(np.complex128) for x in dc]
        assert np.array_equal(bits(got[0]), bits(want.t1)) and np.array_equal(bits(got[1]), bits(want.t2)), i
    for lo, hi in [(0, 5), (5, 13), (13, 32)]:
        sa = qt.CdTensor3(hi - lo, n, p, np.ascontiguousarray(a.t1[:, lo:hi]), np.ascontiguousarray(a.t2[:, lo:hi]))
        c = qt.tprod_fast(sa, b)
        assert np.array_equal(bits(c.t1), bits(want.t1[:, lo:hi])) and np.array_equal(bits(c.t2), bits(want.t2[:, lo:hi]))


# ------------------------------------------------------------------------------
# The warp-specialised stage-2 kernel for whole-slice tiles (qt_gemm.cu
# paired_tiny_ws_kernel: m, s <= 16, n <= 16; config 3): bitwise the
# cp.async-ring kernel's result ($QTB_TINY=0), which the parity tests pin to
# the reference.
TINY_SHAPES = [(16, 16, 16, 4096), (16, 16, 16, 64), (12, 16, 9, 256), (16, 8, 16, 128), (5, 3, 7, 33),
               (1, 1, 1, 6), (16, 16, 16, 1), (9, 40, 13, 4096), (3, 33, 2, 4096)]

_TINY_OFF = """
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import paper_2212_14318_b200 as qt
from test_gpu_small import TINY_SHAPES, tiny_inputs
for k, (m, n, s, p) in enumerate(TINY_SHAPES):
    a, b = tiny_inputs(m, n, s, p, k)
    c = qt.tprod_fast(qt.CdTensor3(m, n, p, a[0], a[1]), qt.CdTensor3(n, s, p, b[0], b[1]))
    np.save({path!r} + f"_{{k}}_1.npy", c.t1); np.save({path!r} + f"_{{k}}_2.npy", c.t2)
print("ok")
"""


def tiny_inputs(m, n, s, p, k):
    a = O.gen_random_tensor(m, n, p, 700 + 2 * k)
    b = O.gen_random_tensor(n, s, p, 701 + 2 * k)
    if k == 3:
        a[1][2, 1, 0] = -np.inf
        b[0][p - 2, 0, 3] = complex(1.0, np.nan)
    return a, b


@pytest.fixture(scope="module")
def tiny_off(tmp_path_factory):
    path = str(tmp_path_factory.mktemp("tiny") / "c")
    env = dict(os.environ, QTB_TINY="0")
    code = _TINY_OFF.format(root=ROOT, tests=os.path.join(ROOT, "tests"), path=path)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]
    return path


@pytest.mark.parametrize("k", range(len(TINY_SHAPES)))
def test_tiny_stage2_bitwise_and_parity(tiny_off, k):
    m, n, s, p = TINY_SHAPES[k]
    a, b = tiny_inputs(m, n, s, p, k)
    c = qt.tprod_fast(qt.CdTensor3(m, n, p, a[0], a[1]), qt.CdTensor3(n, s, p, b[0], b[1]))
    w1 = np.load(tiny_off + f"_{k}_1.npy")
    w2 = np.load(tiny_off + f"_{k}_2.npy")
    assert np.array_equal(bits(c.t1), bits(w1)) and np.array_equal(bits(c.t2), bits(w2)), (m, n, s, p)
    if k != 3 and p <= 256:
        assert O.rel_frob_error((c.t1, c.t2), O.tprod_fast(a, b)) <= 1e-12


def test_random_shapes_against_oracle():
    """Random shapes inside both new kernels' domains (the one-launch cluster
    kernel: p in {2, 4, 8, 16}, m, s <= 32, n <= 64; the tiny-tile K2: m, s <= 16,
    n <= 16, any p), checked against the reference restated (<= 1e-12) and the
    definitional product (<= 1e-11)."""
    rng = np.random.default_rng(20261020)
    L = _native.lib()
    fused = tiny = 0
    for it in range(40):
        if it % 2 == 0:
            m, s = (int(x) for x in rng.integers(1, 33, 2))
            n = int(rng.integers(1, 65))
            p = int(rng.choice([2, 4, 8, 16]))
        else:
            m, n, s = (int(x) for x in rng.integers(1, 17, 3))
            p = int(rng.integers(1, 70))
        fused += L.qt_small_fused(m, n, s, p)
        tiny += 1 if (m <= 16 and s <= 16 and n <= 16 and not L.qt_small_fused(m, n, s, p)) else 0
        a = O.gen_random_tensor(m, n, p, 5000 + it)
        b = O.gen_random_tensor(n, s, p, 6000 + it)
        c = qt.tprod_fast(qt.CdTensor3(m, n, p, a[0], a[1]), qt.CdTensor3(n, s, p, b[0], b[1]))
        got = (c.t1, c.t2)
        assert O.rel_frob_error(got, O.tprod_fast(a, b)) <= 1e-12, (m, n, s, p)
        assert O.rel_frob_error(got, O.tprod_naive(a, b)) <= 1e-11, (m, n, s, p)
    assert fused >= 15 and tiny >= 10
