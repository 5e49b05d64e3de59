"""GPU parity: the sm_100a pipeline (through the C-ABI) against the oracle and
against the reference's own outputs (tests/golden, made from oracle/_ref).

Tolerance (BASELINE.json north_star): relative Frobenius error <= 1e-12 in
fp64 against the reference's FFT-based tprod_fast; the reference tests' own
bars where they are tighter/looser (1e-11 random shapes vs the definitional
product, test_tproduct.cpp:105-112; 1e-13 at p = 1, :100-103).
"""
import numpy as np
import pytest

import oracle as O
import paper_2212_14318_b200 as qt
from paper_2212_14318_b200 import _native
from conftest import RefRng

pytestmark = pytest.mark.gpu

TOL = 1e-12
ROOT_DIR = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))


def as_pair(t):
    return (t.t1, t.t2)


def to_cd(pair):
    p, m, n = pair[0].shape
    return qt.CdTensor3(m, n, p, pair[0], pair[1])


def gpu_tprod(a, b):
    return as_pair(qt.tprod_fast(to_cd(a), to_cd(b)))


def bits_equal(x, y):
    return np.array_equal(np.ascontiguousarray(x).view(np.uint64), np.ascontiguousarray(y).view(np.uint64))


# ----------------------------------------------------- reference test-suite
def test_fast_equals_naive_reference_suite():  # test_tproduct.cpp:88-116
    rng = RefRng(11)
    a, b = rng.tensor(5, 4, 6), rng.tensor(4, 3, 6)
    assert O.rel_frob_error(gpu_tprod(a, b), O.tprod_naive(a, b)) <= 1e-11
    a, b = rng.tensor(2, 3, 1), rng.tensor(3, 2, 1)
    assert O.rel_frob_error(gpu_tprod(a, b), O.tprod_naive(a, b)) <= 1e-13
    for _ in range(60):
        m, n = 1 + rng.next_u64() % 8, 1 + rng.next_u64() % 8
        s, p = 1 + rng.next_u64() % 8, 1 + rng.next_u64() % 12
        a, b = rng.tensor(m, n, p), rng.tensor(n, s, p)
        g = gpu_tprod(a, b)
        assert O.rel_frob_error(g, O.tprod_naive(a, b)) <= 1e-11, (m, n, s, p)
        assert O.rel_frob_error(g, O.tprod_fast(a, b)) <= TOL, (m, n, s, p)
    with pytest.raises(ValueError):
        qt.tprod_fast(to_cd(rng.tensor(2, 2, 2)), to_cd(rng.tensor(3, 2, 2)))


def test_acceptance_criterion_1_on_gpu():  # acceptance.cpp:46-65
    rng = RefRng(20240001)
    worst = 0.0
    for _ in range(100):
        m, n = 1 + rng.next_u64() % 8, 1 + rng.next_u64() % 8
        s, p = 1 + rng.next_u64() % 8, 1 + rng.next_u64() % 12
        a = O.gen_random_tensor(m, n, p, rng.next_u64())
        b = O.gen_random_tensor(n, s, p, rng.next_u64())
        worst = max(worst, O.rel_frob_error(gpu_tprod(a, b), O.tprod_naive(a, b)))
    assert worst <= 1e-11
    a = O.gen_random_tensor(50, 50, 10, 1001)
    b = O.gen_random_tensor(50, 50, 10, 1002)
    assert O.rel_frob_error(gpu_tprod(a, b), O.tprod_naive(a, b)) <= 1e-12


def test_workspace_reuse_bitwise():  # test_tproduct.cpp:118-128
    rng = RefRng(13)
    ws = qt.TProdWorkspace()
    for _ in range(3):
        a, b = to_cd(rng.tensor(4, 3, 8)), to_cd(rng.tensor(3, 5, 8))
        c1 = qt.tprod_fast(a, b, ws)
        c2 = qt.tprod_fast(a, b)
        assert bits_equal(c1.t1, c2.t1) and bits_equal(c1.t2, c2.t2)


@pytest.mark.parametrize("m,n,s,p", [(4, 3, 5, 8), (24, 16, 20, 12), (40, 256, 520, 5), (3, 0, 2, 4)])
def test_workspace_spectra_like_reference(m, n, s, p):
    """qt_tprod_f64_host_spectra (the drop-in with $QTB_DROPIN_FILL_WS=1):
    Â, B̂, Ĉ come back like the reference's ws (tproduct.cpp:80-87) — Â, B̂
    equal the reference's qfft3_conj within 1e-13, Ĉ inverse-transforms to C
    — and C is qt_tprod_f64_host's, bitwise (the int8 shape included)."""
    L = _native.lib()
    a = qt.gen_random_tensor(m, max(n, 1), p, 5) if n else qt.CdTensor3(m, 0, p)
    b = qt.gen_random_tensor(max(n, 1), s, p, 6) if n else qt.CdTensor3(0, s, p)
    c = qt.CdTensor3(m, s, p)
    ah, bh, ch = qt.CdTensor3(m, n, p), qt.CdTensor3(n, s, p), qt.CdTensor3(m, s, p)
    ptr = lambda x: x.ctypes.data
    _native.check(L.qt_tprod_f64_host_spectra(ptr(a.t1), ptr(a.t2), ptr(b.t1), ptr(b.t2), ptr(c.t1), ptr(c.t2), m, n,
                                              s, p, 0, ptr(ah.t1), ptr(ah.t2), ptr(bh.t1), ptr(bh.t2), ptr(ch.t1),
                                              ptr(ch.t2)), "tprod spectra")
    want = qt.tprod_fast(a, b)
    assert bits_equal(c.t1, want.t1) and bits_equal(c.t2, want.t2)
    if n:
        assert O.rel_frob_error((ah.t1, ah.t2), O.qfft3_conj((a.t1, a.t2))) <= 1e-13
        assert O.rel_frob_error((bh.t1, bh.t2), O.qfft3_conj((b.t1, b.t2))) <= 1e-13
        back = qt.qifft3_conj(ch)
        assert bits_equal(back.t1, c.t1) and bits_equal(back.t2, c.t2)
    else:
        assert not np.any(ch.t1) and not np.any(c.t1)


def test_real_inputs_match_per_slice_spectral_product():  # test_tproduct.cpp:130-166
    rng = RefRng(17)
    m, n, s, p = 3, 2, 4, 6
    a = qt.CdTensor3(m, n, p)
    b = qt.CdTensor3(n, s, p)
    a.t1.real = np.array([rng.sym() for _ in range(m * n * p)]).reshape(p, m, n)
    b.t1.real = np.array([rng.sym() for _ in range(n * s * p)]).reshape(p, n, s)
    ah = np.fft.fft(a.t1, axis=0)
    bh = np.fft.fft(b.t1, axis=0)
    want = np.fft.ifft(np.einsum("kij,kjl->kil", ah, bh), axis=0)
    c = qt.tprod_fast(a, b)
    err = np.sqrt(np.sum(np.abs(c.t1 - want) ** 2) + np.sum(np.abs(c.t2) ** 2)) / np.sqrt(np.sum(np.abs(want) ** 2))
    assert err <= 1e-12


def test_identity_and_circular_convolution():  # test_tproduct.cpp:60-86 through the fast path
    rng = RefRng(7)
    t = rng.tensor(3, 4, 6)
    eye = (np.zeros((6, 4, 4), np.complex128), np.zeros((6, 4, 4), np.complex128))
    eye[0][0] = np.eye(4)
    assert O.rel_frob_error(gpu_tprod(t, eye), t) <= 1e-12
    x, y = rng.tensor(1, 1, 5), rng.tensor(1, 1, 5)
    assert O.rel_frob_error(gpu_tprod(x, y), O.tprod_naive(x, y)) <= 1e-13


# --------------------------------------------------------- golden fixtures
def test_golden_small_cases(small_golden):
    g = small_golden
    for k in range(int(g["ncases"])):
        a = (g[f"c{k}_a1"], g[f"c{k}_a2"])
        b = (g[f"c{k}_b1"], g[f"c{k}_b2"])
        got = gpu_tprod(a, b)
        shape = tuple(int(v) for v in g[f"c{k}_shape"])
        assert O.rel_frob_error(got, (g[f"c{k}_fast1"], g[f"c{k}_fast2"])) <= TOL, shape
        assert O.rel_frob_error(got, (g[f"c{k}_naive1"], g[f"c{k}_naive2"])) <= 1e-11, shape
        fa = qt.qfft3_conj(to_cd(a))
        assert O.rel_frob_error(as_pair(fa), (g[f"c{k}_fa1"], g[f"c{k}_fa2"])) <= TOL, shape
        ia = qt.qifft3_conj(to_cd(a))
        assert O.rel_frob_error(as_pair(ia), (g[f"c{k}_ia1"], g[f"c{k}_ia2"])) <= TOL, shape


@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_baseline_config_against_reference_tiles(cfg_golden, c):
    """Full BASELINE config on the GPU; compared with the reference's own output
    on sampled row x column tiles (every 1/2/4/8-way shard boundary row)."""
    g = cfg_golden
    cfg = qt.CONFIGS[c]
    a, b = qt.make_inputs(cfg)
    chk = np.array([np.sum(a.t1.real), np.sum(a.t1.imag), np.sum(a.t2.real), np.sum(a.t2.imag)])
    assert np.array_equal(chk, g[f"cfg{c}_chkA"]), "input generator drifted from the fixture"
    out = qt.tprod_fast(a, b)
    rows, cols, sl = g[f"cfg{c}_rows"], g[f"cfg{c}_cols"], g[f"cfg{c}_slices"]
    t1 = out.t1[:, rows][:, :, cols]
    t2 = out.t2[:, rows][:, :, cols]
    assert O.rel_frob_error((t1[sl], t2[sl]), (g[f"cfg{c}_c1"], g[f"cfg{c}_c2"])) <= TOL
    sums = np.stack([t1.sum(0), t2.sum(0)])
    assert np.linalg.norm(sums - g[f"cfg{c}_sum"]) <= TOL * np.sqrt(np.sum(g[f"cfg{c}_sumsq"])) * np.sqrt(cfg.p)
    sumsq = np.stack([(np.abs(t1) ** 2).sum(0), (np.abs(t2) ** 2).sum(0)])
    assert np.allclose(sumsq, g[f"cfg{c}_sumsq"], rtol=1e-11, atol=0)
    if c == 1:
        full = (g["cfg1_full_fast1"], g["cfg1_full_fast2"])
        assert O.rel_frob_error(as_pair(out), full) <= TOL
        assert O.rel_frob_error(as_pair(out), O.tprod_naive(as_pair(a), as_pair(b))) <= TOL


# ------------------------------------------------------------- edge cases
@pytest.mark.parametrize("m,n,s,p", [
    (1, 1, 1, 1), (3, 5, 2, 1), (4, 4, 4, 2), (7, 3, 9, 3), (5, 6, 7, 5), (8, 8, 8, 7),
    (9, 10, 11, 13), (70, 33, 17, 16), (65, 17, 33, 64), (130, 9, 70, 32), (3, 200, 5, 20),
    (2, 3, 4, 97), (16, 16, 16, 128), (4, 4, 4, 1024), (2, 3, 2, 4096), (1, 1, 1, 8192),
    (1, 2, 1, 10007), (33, 1, 35, 12), (1, 40, 1, 9), (64, 64, 16, 6),
])
def test_shapes_against_oracle(m, n, s, p):
    a = O.gen_random_tensor(m, n, p, 1000 + m)
    b = O.gen_random_tensor(n, s, p, 2000 + s)
    got = gpu_tprod(a, b)
    want = O.tprod_fast(a, b)
    assert O.rel_frob_error(got, want) <= TOL, (m, n, s, p)


def test_degenerate_zero_dims():
    for (m, n, s, p) in [(0, 3, 2, 4), (3, 0, 2, 4), (3, 2, 0, 4)]:
        a = qt.CdTensor3(m, n, p)
        b = qt.CdTensor3(n, s, p)
        if m * n:
            a.t1[...] = 1 + 1j
        c = qt.tprod_fast(a, b)
        assert c.t1.shape == (p, m, s) and not np.any(c.t1) and not np.any(c.t2)
    with pytest.raises(ValueError):
        qt.tprod_fast(qt.CdTensor3(2, 2, 0), qt.CdTensor3(2, 2, 0))  # transform.cpp:152


def test_transform_kats_on_gpu():  # test_transform.cpp:102-168
    tube = qt.CdTensor3(1, 1, 4)
    for r in range(4):
        tube.set_qat(0, 0, r, (0.0, 0.0, float(r + 1), 0.0))
    hat = qt.qfft3_conj(tube)
    want = [(0, 0, -10, 0), (0, 0, 2, -2), (0, 0, 2, 0), (0, 0, 2, 2)]
    for r in range(4):
        assert np.allclose(hat.qat(0, 0, r), want[r], atol=1e-13, rtol=0)
    one = qt.CdTensor3(1, 1, 1)
    one.set_qat(0, 0, 0, (1.0, 2.0, 3.0, 4.0))
    assert qt.qifft3_conj(one).qat(0, 0, 0) == (1.0, -2.0, -3.0, -4.0)
    rng = RefRng(71)
    t = to_cd(rng.tensor(3, 4, 5))
    assert O.rel_frob_error(as_pair(qt.qifft3_conj(qt.qfft3_conj(t))), as_pair(t)) <= 1e-12
    re = qt.CdTensor3(2, 2, 5)
    re.t1.real = np.arange(20).reshape(5, 2, 2) / 7.0
    h = qt.qfft3_conj(re)
    assert np.all(h.t2 == 0)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8, 9, 11, 12, 15, 16, 17, 24, 32, 60, 64, 97, 100, 243, 256,
                               1000, 4096, 7919, 8192, 16384])
def test_transforms_against_oracle(p):
    m, n = (3, 5) if p <= 4096 else (1, 3)
    x = O.gen_random_tensor(m, n, p, 77 + p)
    for gpu_fn, orc_fn in ((qt.qfft3_conj, O.qfft3_conj), (qt.qifft3_conj, O.qifft3_conj)):
        got = as_pair(gpu_fn(to_cd(x)))
        assert O.rel_frob_error(got, orc_fn(x)) <= TOL, p


@pytest.mark.parametrize("p", [1, 2, 3, 5, 8, 16, 24, 32, 64, 97, 128, 256, 512])
def test_routed_transforms_bitwise(p):
    """qt_q{i}fft3_conj_f64_device_routed: frequency rows scattered to (gathered
    from) arbitrary places through per-row pointer tables equal the plain
    transforms bitwise."""
    import torch
    L = _native.lib()
    assert L.qt_fft_routable(p) == 1
    m, n = 7, 9
    x = torch.randn((2, p, m, 2 * n), dtype=torch.float64, device="cuda")
    plain = torch.empty_like(x)
    _native.check(L.qt_qfft3_conj_f64_device(x[0].data_ptr(), x[1].data_ptr(), plain[0].data_ptr(),
                                             plain[1].data_ptr(), m, n, p, None), "qfft3")
    perm = torch.randperm(p).tolist()  # row k lands in slice perm[k] of a scratch tensor
    scat = torch.full_like(x, float("nan"))
    tab = torch.tensor([[scat[pl, perm[k]].data_ptr() for k in range(p)] for pl in (0, 1)], dtype=torch.int64,
                       device="cuda")
    _native.check(L.qt_qfft3_conj_f64_device_routed(x[0].data_ptr(), x[1].data_ptr(), tab[0].data_ptr(),
                                                    tab[1].data_ptr(), m, n, p, None), "qfft3 routed")
    assert torch.equal(scat[:, perm].view(torch.int64), plain.view(torch.int64))
    inv = torch.empty_like(x)
    _native.check(L.qt_qifft3_conj_f64_device(plain[0].data_ptr(), plain[1].data_ptr(), inv[0].data_ptr(),
                                              inv[1].data_ptr(), m, n, p, None), "qifft3")
    inv_r = torch.empty_like(x)
    _native.check(L.qt_qifft3_conj_f64_device_routed(tab[0].data_ptr(), tab[1].data_ptr(), inv_r[0].data_ptr(),
                                                     inv_r[1].data_ptr(), m, n, p, None), "qifft3 routed")
    assert torch.equal(inv_r.view(torch.int64), inv.view(torch.int64))


def test_routed_transforms_reject_two_pass_lengths():
    L = _native.lib()
    assert L.qt_fft_routable(4096) == 0 and L.qt_fft_routable(0) == 0
    import torch
    x = torch.zeros((2, 4096, 1, 2), dtype=torch.float64, device="cuda")
    tab = torch.zeros((2, 4096), dtype=torch.int64, device="cuda")
    assert L.qt_qfft3_conj_f64_device_routed(x[0].data_ptr(), x[1].data_ptr(), tab[0].data_ptr(), tab[1].data_ptr(),
                                             1, 1, 4096, None) == _native.QT_EINVAL


@pytest.mark.parametrize("m,n,s,p,kernels", [(32, 32, 32, 16, 3), (8, 8, 8, 4096, 5)])
def test_small_product_graph_replay(m, n, s, p, kernels):
    """qt_tprod_f64_device records a small product into a CUDA graph on its
    first call and replays it afterwards: every call is bitwise equal to the
    host entry point, a replay reads the buffers' current contents, and it
    still counts its three kernels."""
    import torch
    L = _native.lib()
    dev = torch.device("cuda", 0)
    a = qt.gen_random_tensor(m, n, p, 501)
    b = qt.gen_random_tensor(n, s, p, 502)
    da = [torch.from_numpy(x.view(np.float64)).to(dev) for x in (a.t1, a.t2)]
    db = [torch.from_numpy(x.view(np.float64)).to(dev) for x in (b.t1, b.t2)]
    dc = [torch.empty((p, m, 2 * s), dtype=torch.float64, device=dev) for _ in range(2)]

    def call():
        _native.check(L.qt_tprod_f64_device(da[0].data_ptr(), da[1].data_ptr(), db[0].data_ptr(), db[1].data_ptr(),
                                            dc[0].data_ptr(), dc[1].data_ptr(), m, n, s, p, None), "tprod")
        torch.cuda.synchronize()
        return [x.cpu().numpy().view(np.complex128) for x in dc]

    if L.qt_small_fused(m, n, s, p):  # one launch instead of three (csrc/qt_small.cu)
        kernels = 1
    want = qt.tprod_fast(a, b)
    for i in range(3):  # direct + capture, then replays
        before = L.qt_kernel_launches()
        got = call()
        assert bits_equal(got[0], want.t1) and bits_equal(got[1], want.t2), i
        assert L.qt_kernel_launches() - before == kernels, i
    a2 = qt.gen_random_tensor(m, n, p, 503)  # new contents, same buffers
    da[0].copy_(torch.from_numpy(a2.t1.view(np.float64)))
    da[1].copy_(torch.from_numpy(a2.t2.view(np.float64)))
    got = call()
    want2 = qt.tprod_fast(a2, b)
    assert bits_equal(got[0], want2.t1) and bits_equal(got[1], want2.t2)


def test_graph_cache_many_keys_and_shapes():
    """More than the cache holds (64) distinct (pointers, shape) keys, several
    shapes incl. p = 1 and a prime length, revisited in a different order:
    every call equals the host entry point bitwise."""
    import torch
    L = _native.lib()
    dev = torch.device("cuda", 0)
    shapes = [(5, 3, 4, 1), (6, 4, 5, 7), (9, 8, 7, 12), (4, 6, 3, 97)]
    bufs = []
    for i in range(70):
        m, n, s, p = shapes[i % len(shapes)]
        a = qt.gen_random_tensor(m, n, p, 700 + i)
        b = qt.gen_random_tensor(n, s, p, 800 + i)
        da = [torch.from_numpy(x.view(np.float64)).to(dev) for x in (a.t1, a.t2)]
        db = [torch.from_numpy(x.view(np.float64)).to(dev) for x in (b.t1, b.t2)]
        dc = [torch.empty((p, m, 2 * s), dtype=torch.float64, device=dev) for _ in range(2)]
        bufs.append(((m, n, s, p), a, b, da, db, dc))
    for rnd in range(2):
        order = range(len(bufs)) if rnd == 0 else reversed(range(len(bufs)))
        for i in order:
            (m, n, s, p), a, b, da, db, dc = bufs[i]
            _native.check(L.qt_tprod_f64_device(da[0].data_ptr(), da[1].data_ptr(), db[0].data_ptr(),
                                                db[1].data_ptr(), dc[0].data_ptr(), dc[1].data_ptr(), m, n, s, p,
                                                None), "tprod")
        torch.cuda.synchronize()
        for (m, n, s, p), a, b, da, db, dc in bufs[::7]:
            want = qt.tprod_fast(a, b)
            got = [x.cpu().numpy().view(np.complex128) for x in dc]
            assert bits_equal(got[0], want.t1) and bits_equal(got[1], want.t2), (rnd, m, n, s, p)


# -------------------------------------------------------------- properties
def test_determinism_and_row_shard_invariance():
    """Repeated calls are bitwise identical, and row slabs computed separately
    and stitched equal the full product bitwise (the G-GPU invariance)."""
    from paper_2212_14318_b200 import shard
    a = qt.gen_random_tensor(100, 48, 16, 5)
    b = qt.gen_random_tensor(48, 40, 16, 6)
    c = qt.tprod_fast(a, b)
    c2 = qt.tprod_fast(a, b)
    assert bits_equal(c.t1, c2.t1) and bits_equal(c.t2, c2.t2)
    for world in (2, 3, 8):
        for r in range(world):
            lo, hi = shard.row_slab(a.m, world, r)
            if hi == lo:
                continue
            s1, s2 = shard.take_rows(a.t1, a.t2, lo, hi)
            part = qt.tprod_fast(qt.CdTensor3(hi - lo, a.n, a.p, s1, s2), b)
            assert bits_equal(part.t1, c.t1[:, lo:hi]) and bits_equal(part.t2, c.t2[:, lo:hi])


def test_linearity_at_full_size():
    """Size-independent property at config-2 scale: (A)(B1 + B2) = A B1 + A B2."""
    cfg = qt.CONFIGS[2]
    a, b1 = qt.make_inputs(cfg)
    b2 = qt.gen_tensor(cfg.n, cfg.s, cfg.p, 4242, qt._native.QT_DIST_NORMAL, 1.0)
    bs = qt.CdTensor3(cfg.n, cfg.s, cfg.p, b1.t1 + b2.t1, b1.t2 + b2.t2)
    lhs = qt.tprod_fast(a, bs)
    r1, r2 = qt.tprod_fast(a, b1), qt.tprod_fast(a, b2)
    assert O.rel_frob_error(as_pair(lhs), (r1.t1 + r2.t1, r1.t2 + r2.t2)) <= 1e-13


@pytest.mark.parametrize("m,n,s,p", [(40, 24, 20, 12), (130, 33, 70, 16), (300, 64, 200, 64), (17, 16, 16, 4096),
                                     (64, 256, 512, 4)])
def test_multi_driver_single_device_matches(m, n, s, p):
    """qt_tprod_f64_multi on one device equals the single-GPU host path
    bitwise (the last shape takes the int8 stage 2)."""
    a = qt.gen_random_tensor(m, n, p, 8)
    b = qt.gen_random_tensor(n, s, p, 9)
    c = qt.tprod_fast(a, b)
    cm = qt.tprod_fast_multi(a, b, [0])
    assert bits_equal(c.t1, cm.t1) and bits_equal(c.t2, cm.t2)


def test_long_tube_sharding_bitwise():
    """p = 4096 (four-step split) and a tiny shard still use the same per-tube
    arithmetic: slabs of 1..16 rows stitch to the full result bitwise."""
    from paper_2212_14318_b200 import shard
    a = qt.gen_random_tensor(16, 16, 4096, 41)
    b = qt.gen_random_tensor(16, 16, 4096, 42)
    c = qt.tprod_fast(a, b)
    for world in (2, 16):
        for r in range(world):
            lo, hi = shard.row_slab(16, world, r)
            s1, s2 = shard.take_rows(a.t1, a.t2, lo, hi)
            part = qt.tprod_fast(qt.CdTensor3(hi - lo, 16, 4096, s1, s2), b)
            assert bits_equal(part.t1, c.t1[:, lo:hi]) and bits_equal(part.t2, c.t2[:, lo:hi])


# ------------------------------------------------ GPU definitional product
def test_gpu_naive_reference_kats():  # test_tproduct.cpp:60-86 through the GPU tprod_naive
    rng = RefRng(7)
    a, b = rng.tensor(3, 2, 1), rng.tensor(2, 4, 1)
    c = as_pair(qt.tprod_naive(to_cd(a), to_cd(b)))
    w1 = a[0][0] @ b[0][0] - a[1][0] @ np.conj(b[1][0])
    w2 = a[0][0] @ b[1][0] + a[1][0] @ np.conj(b[0][0])
    assert np.sqrt(np.sum(np.abs(c[0][0] - w1) ** 2) + np.sum(np.abs(c[1][0] - w2) ** 2)) <= 1e-14
    t = rng.tensor(3, 4, 6)
    eye = (np.zeros((6, 4, 4), np.complex128), np.zeros((6, 4, 4), np.complex128))
    eye[0][0] = np.eye(4)
    assert O.rel_frob_error(as_pair(qt.tprod_naive(to_cd(t), to_cd(eye))), t) <= 1e-12
    with pytest.raises(ValueError):
        qt.tprod_naive(to_cd(a), to_cd(rng.tensor(3, 2, 1)))


@pytest.mark.parametrize("m,n,s,p", [(5, 4, 3, 6), (1, 1, 1, 5), (8, 8, 8, 12), (33, 17, 40, 7), (70, 9, 20, 4),
                                     (3, 3, 3, 1), (2, 0, 3, 4)])
def test_gpu_naive_against_oracle_naive(m, n, s, p):
    a = O.gen_random_tensor(m, max(n, 1), p, 500 + m)
    b = O.gen_random_tensor(max(n, 1), s, p, 600 + s)
    if n == 0:
        a = (a[0][:, :, :0], a[1][:, :, :0])
        b = (b[0][:, :0, :], b[1][:, :0, :])
        got = as_pair(qt.tprod_naive(to_cd(a) if m else qt.CdTensor3(m, 0, p), qt.CdTensor3(0, s, p)))
        assert not np.any(got[0]) and not np.any(got[1])
        return
    got = as_pair(qt.tprod_naive(to_cd(a), to_cd(b)))
    assert O.rel_frob_error(got, O.tprod_naive(a, b)) <= 1e-13


def test_gpu_naive_equals_fast_full_config3():
    """Full-tensor check of the FFT path against the O(p^2) definitional
    product on the GPU at BASELINE config 3 (p = 4096, 16 m n s p^2 = 4.4e12)."""
    a, b = qt.make_inputs(qt.CONFIGS[3])
    fast = qt.tprod_fast(a, b)
    naive = qt.tprod_naive(a, b)
    assert O.rel_frob_error(as_pair(fast), as_pair(naive)) <= 1e-12


def test_multi_driver_before_torch_import_keeps_torch_importable():
    """The C driver must not load a second libnccl.so.2 that shadows torch's
    (regression: system NCCL 2.27 loaded first broke `import torch`)."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r)\n"
            "import paper_2212_14318_b200 as qt\n"
            "a = qt.gen_random_tensor(8, 4, 4, 1); b = qt.gen_random_tensor(4, 4, 4, 2)\n"
            "c = qt.tprod_fast_multi(a, b, [0])\n"
            "import torch; assert torch.cuda.is_available(); print('ok')\n") % ROOT_DIR
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_concurrent_host_calls_are_reentrant_and_bitwise():
    """the drop-in must be reentrant.  Several host threads call
    tprod_fast at once (per-thread streams, stream-ordered workspace, shared
    pinned arena and twiddle cache); each result equals its sequential twin."""
    import threading
    shapes = [(40, 24, 30, 16), (300, 64, 200, 32), (16, 16, 16, 4096), (5, 4, 3, 7), (260, 70, 130, 64),
              (33, 17, 40, 12), (64, 256, 512, 8), (150, 288, 520, 5)]  # the last two take the int8 stage 2
    ins = [(qt.gen_random_tensor(m, n, p, 10 + i), qt.gen_random_tensor(n, s, p, 20 + i))
           for i, (m, n, s, p) in enumerate(shapes)]
    want = [qt.tprod_fast(a, b) for a, b in ins]
    got = [None] * len(ins)
    errors = []

    def run(i):
        try:
            for _ in range(3):
                got[i] = qt.tprod_fast(*ins[i])
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in range(len(ins))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for w, g in zip(want, got):
        assert bits_equal(w.t1, g.t1) and bits_equal(w.t2, g.t2)
