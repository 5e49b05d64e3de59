"""GPU parity of the exact int8 (Ozaki-II / CRT) stage 2 — csrc/qt_ozaki.cu.

The product is evaluated exactly in integers and rounded once, so besides the
1e-12 bar of BASELINE.json against the reference's tprod_fast (and its 1e-11
bar against the definitional product, test_tproduct.cpp:105-112) it must be
(a) bitwise independent of batching, row slabs and column chunks, and (b) at
least as accurate as the fp64 DMMA path against a long-double truth.
"""
import numpy as np
import pytest

import oracle as O
import paper_2212_14318_b200 as qt
from paper_2212_14318_b200 import _native

pytestmark = pytest.mark.gpu

DMMA, INT8 = 0, 1


def bits_equal(x, y):
    return np.array_equal(np.ascontiguousarray(x).view(np.uint64), np.ascontiguousarray(y).view(np.uint64))


def torch_cuda():
    import torch
    return torch


def spectral(ah, bh, m, n, s, p, algo, rows=None, cols=None):
    """Stage 2 through qt_spectral_product_f64_device_ld_algo; rows/cols select
    a row slab of Â / column chunk of B̂ (written into the full Ĉ)."""
    torch = torch_cuda()
    L = _native.lib()
    c = torch.zeros((2, p, m, s), dtype=torch.complex128, device="cuda")
    r0, r1 = rows if rows else (0, m)
    c0, c1 = cols if cols else (0, s)
    a = ah[:, :, r0:r1].contiguous()
    b = bh[:, :, :, c0:c1].contiguous()
    cc = torch.zeros((2, p, r1 - r0, s), dtype=torch.complex128, device="cuda")
    off = 16 * c0
    _native.check(L.qt_spectral_product_f64_device_ld_algo(
        a[0].data_ptr(), a[1].data_ptr(), b[0].data_ptr(), b[1].data_ptr(), cc[0].data_ptr() + off,
        cc[1].data_ptr() + off, r1 - r0, n, c1 - c0, p, c1 - c0, s, n * (c1 - c0), (r1 - r0) * s, algo, None),
        "spectral")
    c[:, :, r0:r1] = cc
    torch.cuda.synchronize()
    return c


def random_spectral(m, n, s, p, seed):
    torch = torch_cuda()
    g = torch.Generator(device="cuda").manual_seed(seed)
    ah = torch.randn((2, p, m, n), dtype=torch.complex128, device="cuda", generator=g)
    bh = torch.randn((2, p, n, s), dtype=torch.complex128, device="cuda", generator=g)
    return ah, bh


def reference_spectral(ah, bh):
    """SURVEY §8(a) paired form in numpy float64 (complex128 matmul)."""
    A1, A2 = ah[0].cpu().numpy(), ah[1].cpu().numpy()
    B1, B2 = bh[0].cpu().numpy(), bh[1].cpu().numpy()
    p = A1.shape[0]
    C1 = np.empty((p, A1.shape[1], B1.shape[2]), np.complex128)
    C2 = np.empty_like(C1)
    for k in range(p):
        sk = (p - k) % p
        C1[k] = A1[k] @ B1[k] - np.conj(A2[sk]) @ B2[k]
        C2[k] = np.conj(A1[sk]) @ B2[k] + A2[k] @ B1[k]
    return C1, C2


def rel(x, y):
    """Relative Frobenius error, computed on values normalised by max |y| (so
    extreme magnitudes neither overflow nor underflow when squared)."""
    sc = max(float(np.max(np.abs(b))) for b in y) or 1.0
    return float(np.sqrt(sum(np.sum(np.abs(a / sc - b / sc) ** 2) for a, b in zip(x, y)) /
                         sum(np.sum(np.abs(b / sc) ** 2) for b in y)))


# ---------------------------------------------------------------- algorithm
def test_algorithm_choice_depends_on_n_and_s_only():
    L = _native.lib()
    assert L.qt_gemm_algo(2048, 2048, 2048, 32) == INT8      # config 5
    assert L.qt_gemm_algo(7, 2048, 2048, 32) == INT8         # any row slab of it
    assert L.qt_gemm_algo(1080, 1920, 64, 64) == DMMA        # config 4: narrow output
    assert L.qt_gemm_algo(256, 256, 256, 64) == DMMA         # config 2: too small to amortise
    assert L.qt_gemm_algo(16, 16, 16, 4096) == DMMA          # config 3
    assert L.qt_gemm_algo(32, 32, 32, 16) == DMMA            # config 1
    assert L.qt_gemm_algo(64, 300, 512, 8) == DMMA           # n % 32 != 0


@pytest.mark.parametrize("m,n,s,p", [(1, 32, 1, 5), (2, 32, 2, 3), (4, 64, 4, 1), (64, 96, 80, 8),
                                     (130, 256, 70, 7), (200, 64, 300, 9), (129, 288, 131, 2)])
def test_int8_spectral_matches_fp64(m, n, s, p):
    """Forced int8 path on ragged / odd-p / tiny shapes against numpy fp64 and
    against the DMMA path (both ~1e-16; bar 1e-13)."""
    ah, bh = random_spectral(m, n, s, p, 5 + m + p)
    c8 = spectral(ah, bh, m, n, s, p, INT8)
    cd = spectral(ah, bh, m, n, s, p, DMMA)
    ref = reference_spectral(ah, bh)
    got8 = (c8[0].cpu().numpy(), c8[1].cpu().numpy())
    gotd = (cd[0].cpu().numpy(), cd[1].cpu().numpy())
    assert rel(got8, ref) <= 1e-13
    assert rel(got8, gotd) <= 1e-13


def test_int8_more_accurate_than_fp64_gemm():
    """Against a long-double evaluation the exact-integer product's error is
    no larger than the fp64 DMMA product's (both ~1e-16)."""
    m, n, s, p = 48, 512, 40, 4
    ah, bh = random_spectral(m, n, s, p, 77)
    c8 = spectral(ah, bh, m, n, s, p, INT8)
    cd = spectral(ah, bh, m, n, s, p, DMMA)
    A = [x.cpu().numpy() for x in ah]
    B = [x.cpu().numpy() for x in bh]
    ld = np.longdouble

    def cmm(x, y):  # complex matmul in long double
        xr, xi, yr, yi = (v.astype(ld) for v in (x.real, x.imag, y.real, y.imag))
        return xr @ yr - xi @ yi, xr @ yi + xi @ yr

    err8 = errd = norm = 0.0
    for k in range(p):
        sk = (p - k) % p
        t1 = cmm(A[0][k], B[0][k])
        t2 = cmm(np.conj(A[1][sk]), B[1][k])
        t3 = cmm(np.conj(A[0][sk]), B[1][k])
        t4 = cmm(A[1][k], B[0][k])
        c1 = (t1[0] - t2[0], t1[1] - t2[1])
        c2 = (t3[0] + t4[0], t3[1] + t4[1])
        for got, sq in ((c8, "e8"), (cd, "ed")):
            g1, g2 = got[0][k].cpu().numpy(), got[1][k].cpu().numpy()
            e = (np.sum((g1.real - c1[0]) ** 2 + (g1.imag - c1[1]) ** 2) +
                 np.sum((g2.real - c2[0]) ** 2 + (g2.imag - c2[1]) ** 2))
            if sq == "e8":
                err8 += float(e)
            else:
                errd += float(e)
        norm += float(np.sum(c1[0] ** 2 + c1[1] ** 2) + np.sum(c2[0] ** 2 + c2[1] ** 2))
    e8, ed = np.sqrt(err8 / norm), np.sqrt(errd / norm)
    assert e8 <= 5e-16 and e8 <= ed, (e8, ed)


# --------------------------------------------------------- exactness/bitwise
def test_int8_row_slabs_bitwise_and_column_chunks_accurate():
    """Row slabs of Â use the same per-row scalings and the same balancing of
    the contraction index (from B̂ alone): bitwise equal to the full product.
    A column chunk of B̂ balances over its own columns, so it is equally
    accurate, not bitwise equal."""
    m, n, s, p = 150, 128, 300, 6
    ah, bh = random_spectral(m, n, s, p, 3)
    full = spectral(ah, bh, m, n, s, p, INT8)
    for rows in ((0, 64), (64, 101), (101, 150)):
        part = spectral(ah, bh, m, n, s, p, INT8, rows=rows)
        assert bits_equal(part[:, :, rows[0]:rows[1]].cpu().numpy(), full[:, :, rows[0]:rows[1]].cpu().numpy())
    ref = reference_spectral(ah, bh)
    for cols in ((0, 128), (128, 137), (137, 300)):
        part = spectral(ah, bh, m, n, s, p, INT8, cols=cols).cpu().numpy()
        got = (part[0][..., cols[0]:cols[1]], part[1][..., cols[0]:cols[1]])
        want = (ref[0][..., cols[0]:cols[1]], ref[1][..., cols[0]:cols[1]])
        assert rel(got, want) <= 1e-13


def test_int8_batching_is_bitwise_invariant(monkeypatch):
    m, n, s, p = 96, 256, 260, 7
    ah, bh = random_spectral(m, n, s, p, 4)
    ref = spectral(ah, bh, m, n, s, p, INT8).cpu().numpy()
    monkeypatch.setenv("QTB_OZAKI_WS_MB", "1")   # 2 frequency slots per batch
    monkeypatch.setenv("QTB_OZAKI_B_MB", "1")    # B' rebuilt per batch
    got = spectral(ah, bh, m, n, s, p, INT8).cpu().numpy()
    assert bits_equal(got, ref)


@pytest.mark.parametrize("bad", [float("nan"), float("inf"), -float("inf")])
@pytest.mark.parametrize("where", ["a", "b"])
def test_int8_nonfinite_inputs_fall_back_to_fp64(bad, where):
    """Integers cannot carry inf/nan: the int8 path flags them and the DMMA
    kernels recompute the product, so the result equals the fp64 path's."""
    m, n, s, p = 40, 64, 36, 4
    ah, bh = random_spectral(m, n, s, p, 9)
    if where == "a":
        ah[1, 2, 5, 7] = bad
    else:
        bh[0, 1, 9, 3] = bad
    c8 = spectral(ah, bh, m, n, s, p, INT8).cpu().numpy()
    cd = spectral(ah, bh, m, n, s, p, DMMA).cpu().numpy()
    assert bits_equal(c8, cd)


def test_int8_rejects_unsupported_contraction():
    m, n, s, p = 8, 48, 8, 2  # n % 32 != 0
    ah, bh = random_spectral(m, n, s, p, 1)
    with pytest.raises(ValueError):
        spectral(ah, bh, m, n, s, p, INT8)


# ----------------------------------------------------------- full products
@pytest.mark.parametrize("m,n,s,p", [(40, 256, 520, 5), (130, 288, 512, 4)])
def test_int8_tprod_against_reference_oracle(m, n, s, p):
    """Shapes that select the int8 path by themselves (n >= 256, n s >= 2^17), end to end
    through tprod_fast against the reference restatement (bar 1e-12)."""
    assert _native.lib().qt_gemm_algo(m, n, s, p) == INT8
    a = qt.gen_random_tensor(m, n, p, 21)
    b = qt.gen_random_tensor(n, s, p, 22)
    c = qt.tprod_fast(a, b)
    ref = O.tprod_fast((a.t1, a.t2), (b.t1, b.t2))
    assert O.rel_frob_error((c.t1, c.t2), ref) <= 1e-12


def test_int8_host_slab_stream_bitwise_equals_device_path():
    """A >= 128 MB int8 product takes the row-slab streaming host path
    (resident B' residues); it must equal the device-resident path bitwise."""
    torch = torch_cuda()
    m, n, s, p = 256, 256, 512, 64
    a = qt.gen_random_tensor(m, n, p, 31)
    b = qt.gen_random_tensor(n, s, p, 32)
    host = qt.tprod_fast(a, b)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    c1 = torch.empty((p, m, s), dtype=torch.complex128, device="cuda")
    c2 = torch.empty_like(c1)
    qt.tprod_fast_device(dev(a.t1), dev(a.t2), dev(b.t1), dev(b.t2), c1, c2, m, n, s, p)
    torch.cuda.synchronize()
    assert bits_equal(host.t1, c1.cpu().numpy()) and bits_equal(host.t2, c2.cpu().numpy())


# ------------------------------------------------ sharded drivers
def test_int8_multi_driver_single_device_bitwise():
    m, n, s, p = 130, 256, 520, 4
    a = qt.gen_random_tensor(m, n, p, 51)
    b = qt.gen_random_tensor(n, s, p, 52)
    c = qt.tprod_fast(a, b)
    cm = qt.tprod_fast_multi(a, b, [0])
    assert bits_equal(c.t1, cm.t1) and bits_equal(c.t2, cm.t2)


# ------------------------------------------------------------ magnitudes
@pytest.mark.parametrize("sa,sb", [(2.0 ** 600, 2.0 ** -600), (2.0 ** -500, 2.0 ** -500), (2.0 ** 900, 2.0 ** -1000),
                                   (2.0 ** -1030, 2.0 ** 40)])
def test_int8_extreme_magnitudes_match_fp64(sa, sb):
    """Row/column scaling covers the whole fp64 exponent range (exponents
    outside +-1022 take the ldexp path; subnormal inputs and results)."""
    m, n, s, p = 20, 64, 24, 3
    ah, bh = random_spectral(m, n, s, p, 61)
    ah = ah * sa
    bh = bh * sb
    c8 = spectral(ah, bh, m, n, s, p, INT8)
    cd = spectral(ah, bh, m, n, s, p, DMMA)
    x8 = (c8[0].cpu().numpy(), c8[1].cpu().numpy())
    xd = (cd[0].cpu().numpy(), cd[1].cpu().numpy())
    assert all(np.isfinite(v).all() for v in x8)
    ref = reference_spectral(ah, bh)
    assert rel(x8, xd) <= 1e-13 or rel(x8, ref) <= 1e-13


def test_int8_zero_rows_and_columns():
    m, n, s, p = 24, 64, 30, 4
    ah, bh = random_spectral(m, n, s, p, 62)
    ah[0, :, 3, :] = 0      # row 3 of every A1 slice
    ah[1, :, 3, :] = 0
    bh[:, :, :, 7] = 0      # column 7 of every B slice
    c8 = spectral(ah, bh, m, n, s, p, INT8).cpu().numpy()
    cd = spectral(ah, bh, m, n, s, p, DMMA).cpu().numpy()
    assert np.all(c8[..., 7] == 0)
    ref = reference_spectral(ah, bh)
    assert rel((c8[0], c8[1]), ref) <= 1e-13
    assert rel((c8[0], c8[1]), (cd[0], cd[1])) <= 1e-13


def test_int8_random_shape_sweep():
    """Seeded sweep of ragged shapes (n a multiple of 32; odd and even p;
    m, s off every tile multiple; multi-batch budgets) against the fp64 path."""
    import os
    rng = np.random.default_rng(2024)
    for it in range(14):
        m = int(rng.integers(1, 300))
        n = 32 * int(rng.integers(1, 12))
        s = int(rng.integers(1, 300))
        p = int(rng.integers(1, 14))
        ah, bh = random_spectral(m, n, s, p, 100 + it)
        if it % 3 == 0:
            os.environ["QTB_OZAKI_WS_MB"] = "1"
        try:
            c8 = spectral(ah, bh, m, n, s, p, INT8)
        finally:
            os.environ.pop("QTB_OZAKI_WS_MB", None)
        cd = spectral(ah, bh, m, n, s, p, DMMA)
        e = rel((c8[0].cpu().numpy(), c8[1].cpu().numpy()), (cd[0].cpu().numpy(), cd[1].cpu().numpy()))
        assert e <= 1e-13, (m, n, s, p, e)


def test_int8_maximum_contraction_length():
    """n = 8192 (K' = 4n = 32768: the largest int8 contraction, 255^2 K' < 2^31)
    with near-maximal residues, against the fp64 path."""
    m, n, s, p = 6, 8192, 10, 2
    ah, bh = random_spectral(m, n, s, p, 71)
    c8 = spectral(ah, bh, m, n, s, p, INT8)
    cd = spectral(ah, bh, m, n, s, p, DMMA)
    e = rel((c8[0].cpu().numpy(), c8[1].cpu().numpy()), (cd[0].cpu().numpy(), cd[1].cpu().numpy()))
    assert e <= 1e-13, e
    with pytest.raises(ValueError):  # n = 8224 exceeds the exact-accumulation bound
        spectral(*random_spectral(2, 8224, 2, 1, 1), 2, 8224, 2, 1, INT8)


# ------------------------------------------------ compact slot ranges (N > 1)
def slots_product(ah, bh, m, n, s, p, t0, t1, flag=None):
    """qt_int8_slots_* on the compact slot range [t0, t1) of frequency-ordered
    Â/B̂; returns the compact Ĉ (slot order) and the non-finite flag."""
    import ctypes
    from paper_2212_14318_b200 import shard
    torch = torch_cuda()
    L = _native.lib()
    idx = torch.tensor([shard.slot_freq(p, t) for t in range(t0, t1)], device="cuda")
    a = ah[:, idx].contiguous()
    b = bh[:, idx].contiguous()
    c = torch.zeros((2, t1 - t0, m, s), dtype=torch.complex128, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda") if flag is None else flag
    h = ctypes.c_void_p()
    _native.check(L.qt_int8_slots_create(b[0].data_ptr(), b[1].data_ptr(), n, s, p, t0, t1 - t0, flag.data_ptr(), None,
                                         ctypes.byref(h)), "slots create")
    _native.check(L.qt_int8_slots_multiply(h, a[0].data_ptr(), a[1].data_ptr(), m, c[0].data_ptr(), c[1].data_ptr(),
                                           None), "slots multiply")
    _native.check(L.qt_int8_slots_destroy(h, None), "slots destroy")
    torch.cuda.synchronize()
    return c, int(flag.item())


@pytest.mark.parametrize("m,n,s,p", [(70, 64, 300, 5), (40, 96, 130, 8), (33, 32, 17, 2), (20, 64, 40, 1),
                                     (300, 128, 256, 7)])
def test_int8_slot_ranges_bitwise(m, n, s, p):
    """Every slot of a compact range equals the same frequency of the full
    int8 product bitwise, for every range of every decomposition."""
    from paper_2212_14318_b200 import shard
    L = _native.lib()
    assert [L.qt_slot_frequency(p, t) for t in range(p + 1)] == [shard.slot_freq(p, t) for t in range(p)] + [-1]
    ah, bh = random_spectral(m, n, s, p, 70 + p)
    full = spectral(ah, bh, m, n, s, p, INT8).cpu().numpy()
    ranges = {r for G in (1, 2, 3, 5) for r in shard.slot_ranges(p, G) if r[1] > r[0]}
    for t0, t1 in sorted(ranges):
        c, flag = slots_product(ah, bh, m, n, s, p, t0, t1)
        assert flag == 0
        got = c.cpu().numpy()
        for t in range(t0, t1):
            k = shard.slot_freq(p, t)
            assert bits_equal(got[:, t - t0], full[:, k]), (t0, t1, t)


def test_int8_slot_ranges_nonfinite_and_rejection():
    import ctypes
    torch = torch_cuda()
    L = _native.lib()
    m, n, s, p = 30, 64, 50, 6
    ah, bh = random_spectral(m, n, s, p, 81)
    bh[0, 2, 3, 4] = float("nan")  # frequency 2 = slot 2
    _, flag = slots_product(ah, bh, m, n, s, p, 2, 4)
    assert flag != 0
    _, flag = slots_product(ah, bh, m, n, s, p, 0, 2)
    assert flag == 0
    ah2, bh2 = random_spectral(m, n, s, p, 82)
    ah2[1, 5, 0, 0] = float("inf")  # frequency 5 = slot 1 (partner of slot 0)
    _, flag = slots_product(ah2, bh2, m, n, s, p, 0, 2)
    assert flag != 0
    f = torch.zeros(1, dtype=torch.int32, device="cuda")
    h = ctypes.c_void_p()
    for t0, ns in [(1, 2), (0, 3), (2, 5), (-2, 2), (0, 0)]:  # splits a pair / leaves [0, p)
        assert L.qt_int8_slots_create(bh[0].data_ptr(), bh[1].data_ptr(), n, s, p, t0, ns, f.data_ptr(), None,
                                      ctypes.byref(h)) == _native.QT_EINVAL, (t0, ns)
    # p = 6: slots 4 (frequency 0) and 5 (frequency 3) are self-paired, so [5, 6) is a valid range
    ah3, bh3 = random_spectral(m, n, s, p, 83)
    c, flag = slots_product(ah3, bh3, m, n, s, p, 5, 6)
    full = spectral(ah3, bh3, m, n, s, p, INT8).cpu().numpy()
    assert flag == 0 and bits_equal(c.cpu().numpy()[:, 0], full[:, 3])


@pytest.mark.parametrize("env", [{"QTB_OZAKI_SHAREX": "0"}, {"QTB_RESB_COLS": "32"}, {"QTB_OZAKI_2SM": "0"}])
def test_implementation_switches_bitwise(tmp_path, env):
    """The int8 stage 2 is the same integer computation whatever the layout
    switch: shared X' within a frequency pair on/off, 16- or 32-column B'
    residue tiles, CTA-pair or 1-CTA GEMM — bitwise equal outputs (the
    switches are read once per process, so the other setting runs in a
    subprocess: tools/sharex_check.py)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "ref.npz")
    tool = os.path.join(root, "tools", "sharex_check.py")
    r1 = subprocess.run([sys.executable, tool, out], capture_output=True, text=True, cwd=root, timeout=600)
    assert r1.returncode == 0 and "saved" in r1.stdout, r1.stderr[-2000:]
    r2 = subprocess.run([sys.executable, tool, out], capture_output=True, text=True, cwd=root, timeout=600,
                        env={**os.environ, **env})
    assert r2.returncode == 0, r2.stderr[-2000:]
    lines = [x for x in r2.stdout.splitlines() if x.strip()]
    assert len(lines) == 5 and all(x.endswith("bitwise equal") for x in lines), r2.stdout


# ------------------------------------------------ badly scaled contractions
@pytest.mark.parametrize("case", ["col1e8", "col1e4", "logu_pair", "logu_a", "logu_b_rows", "one_elem"])
def test_int8_badly_scaled_contraction_index(case):
    """A contraction index scaled up in A and down in B (1e8, 1e4, 2^U(-30,30)
    on every index), one-sided scalings and a single huge entry, at a shape
    that selects the int8 stage 2 (64 x 512 x 256, p = 8): tprod_fast stays
    within the north_star's 1e-12 of the reference's tprod_fast (per-element
    fp64 MACs, tproduct.cpp:57-71).  Paired scalings are removed exactly by
    the power-of-two balancing (no pair needs the fp64 fallback)."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "guard_check", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools",
                                    "guard_check.py"))
    gc = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gc)
    L = _native.lib()
    m, n, s, p = 64, 512, 256, 8
    assert L.qt_gemm_algo(m, n, s, p) == INT8
    a, b = gc.scaled_inputs(case, m, n, s, p)
    f0 = L.qt_int8_guard_fallbacks()
    c = qt.tprod_fast(a, b)
    fb = L.qt_int8_guard_fallbacks() - f0
    err = O.rel_frob_error((c.t1, c.t2), O.tprod_fast((a.t1, a.t2), (b.t1, b.t2)))
    assert err <= 1e-12, (case, err, fb)
    if case in ("col1e8", "col1e4", "logu_pair"):
        assert fb == 0, (case, fb)


def test_int8_guard_certifies_wellscaled_products():
    """Well-scaled data (the BASELINE distributions) never needs the fp64
    fallback: the certified bound is ~1e-14 against the 2^-42 tolerance."""
    L = _native.lib()
    f0 = L.qt_int8_guard_fallbacks()
    for (m, n, s, p), seed in (((40, 256, 520, 5), 1), ((64, 1024, 256, 4), 2), ((8, 8192, 128, 2), 3)):
        a = qt.gen_random_tensor(m, n, p, seed)
        b = qt.gen_random_tensor(n, s, p, seed + 10)
        qt.tprod_fast(a, b)
    ah, bh = random_spectral(70, 2048, 512, 4, 9)
    spectral(ah, bh, 70, 2048, 512, 4, INT8)
    assert L.qt_int8_guard_fallbacks() == f0


def _guard_run(env):
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "guard_check.py")], capture_output=True,
                       text=True, cwd=root, timeout=900, env={**os.environ, **env})
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_int8_guard_without_balancing_falls_back():
    """With the balancing switched off ($QTB_OZAKI_BALANCE=0) the per-row /
    per-column scalings alone lose the low-order bits of a 1e8-scaled index
    (~1e-8 error): the guard must reject those pairs and the fp64
    kernels recompute them, keeping every case within 1e-12."""
    out = _guard_run({"QTB_OZAKI_BALANCE": "0"})
    for case in ("plain", "col1e4", "col1e8", "logu_pair", "logu_a", "logu_b_rows", "one_elem"):
        assert out[case]["err"] <= 1e-12, (case, out[case])
    assert out["plain"]["fallbacks"] == 0
    assert out["col1e8"]["fallbacks"] > 0 and out["logu_pair"]["fallbacks"] > 0


def test_int8_guard_forced_fallback_is_the_dmma_product():
    """$QTB_OZAKI_GUARD=force rejects every pair: the int8 call's result is then
    the fp64 DMMA product, bitwise (the fallback recomputes whole pairs)."""
    out = _guard_run({"QTB_OZAKI_GUARD": "force"})
    assert out["forced_bitwise_dmma"] is True
    assert out["plain"]["fallbacks"] > 0 and out["plain"]["err"] <= 1e-12


@pytest.mark.parametrize("case", ["col1e8", "one_elem"])
def test_int8_guard_host_streaming_and_freq_parallel(case):
    """Badly scaled inputs through the other int8 drivers: the host C-ABI path
    that streams A in row slabs against resident B' (each slab's pairs
    certified on their own) against the GPU definitional product, and the
    frequency-parallel split (4 ranks emulated; each slot certified by its
    owner over all rows) bitwise against the one-GPU product."""
    import importlib.util
    import os
    import torch
    from paper_2212_14318_b200 import distributed
    spec = importlib.util.spec_from_file_location(
        "guard_check", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools",
                                    "guard_check.py"))
    gc = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gc)
    m, n, s, p = 512, 512, 256, 16  # >= 128 MB: the host call streams row slabs
    assert _native.lib().qt_gemm_algo(m, n, s, p) == INT8
    a, b = gc.scaled_inputs(case, m, n, s, p, seed=9)
    c = qt.tprod_fast(a, b)
    naive = qt.tprod_naive(a, b)
    assert O.rel_frob_error((c.t1, c.t2), (naive.t1, naive.t2)) <= 1e-12
    m2 = 96
    a2 = qt.CdTensor3(m2, n, p, np.ascontiguousarray(a.t1[:, :m2]), np.ascontiguousarray(a.t2[:, :m2]))
    want = qt.tprod_fast(a2, b)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.float64)).cuda()
    c1 = torch.empty((p, m2, 2 * s), dtype=torch.float64, device="cuda")
    c2 = torch.empty_like(c1)
    distributed.emulate_freq(4, dev(a2.t1), dev(a2.t2), dev(b.t1), dev(b.t2), c1, c2, m2, n, s, p)
    torch.cuda.synchronize()
    assert bits_equal(c1.cpu().numpy().view(np.complex128), want.t1)
    assert bits_equal(c2.cpu().numpy().view(np.complex128), want.t2)
