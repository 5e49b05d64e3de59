"""CPU: pin the oracle (oracle/qt_oracle.c) before trusting it.

1. The known answers of the reference's own test-suite (file:line cited per test).
2. Bitwise equality with the reference's own outputs: the committed fixtures in
   tests/golden/ (generated from oracle/_ref by tests/golden/make_golden.py), and
   live against oracle/_ref when it is built.
"""
import numpy as np
import pytest

import oracle as O
from conftest import RefRng


def cvec(*vals):
    return np.array(vals, np.complex128)


def bits_equal(x, y):
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y)
    return x.shape == y.shape and np.array_equal(x.view(np.uint64), y.view(np.uint64))


def qerr(a, b):
    return np.sqrt(np.sum(np.abs(np.asarray(a) - np.asarray(b)) ** 2))


# ---------------------------------------------------------- test_transform.cpp
def test_direct_dft_pinned_vectors():  # test_transform.cpp:41-57
    y = O.dft_vec_naive(cvec(1, 0, 0, 0))
    assert np.all(np.abs(y - 1) <= 1e-15)
    got = O.dft_vec_naive(cvec(1, 2, 3, 4))
    want = cvec(10, -2 + 2j, -2, -2 - 2j)
    assert np.all(np.abs(got - want) <= 1e-14)
    yc = O.dft_vec_naive(np.full(5, 3 - 1j))
    assert abs(yc[0] - (15 - 5j)) <= 1e-13
    assert np.all(np.abs(yc[1:]) <= 1e-13)
    with pytest.raises(O.OracleError):
        O.dft_vec_naive(np.zeros(0, np.complex128))


def test_fft_awkward_lengths():  # test_transform.cpp:59-70
    f = O.fft_vec(cvec(1, 1))
    assert f[0] == 2 and abs(f[1]) <= 1e-15
    rng = RefRng(51)
    for n in (1, 2, 3, 5, 7, 12, 16, 27, 100, 97):
        x = rng.sym(2 * n).view(np.complex128)
        a, b = O.fft_vec(x), O.dft_vec_naive(x)
        assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-12
    with pytest.raises(O.OracleError):
        O.fft_vec(np.zeros(0, np.complex128))


def test_fft_round_trip_and_linearity():  # test_transform.cpp:72-100
    rng = RefRng(53)
    x = rng.sym(24).view(np.complex128)
    assert np.linalg.norm(O.ifft_vec(O.fft_vec(x)) - x) / np.linalg.norm(x) <= 1e-13
    for n in (4, 9, 14):
        v = rng.sym(2 * n).view(np.complex128)
        assert np.linalg.norm(O.fft_vec(O.ifft_vec(v)) - v) / np.linalg.norm(v) <= 1e-13
    rng = RefRng(57)
    n = 24
    x = rng.sym(2 * n).view(np.complex128).copy()
    y = rng.sym(2 * n).view(np.complex128).copy()
    a = complex(*rng.sym(2))
    b = complex(*rng.sym(2))
    fl = O.fft_vec(a * x + b * y)
    want = a * O.fft_vec(x) + b * O.fft_vec(y)
    assert np.linalg.norm(fl - want) / np.linalg.norm(want) <= 1e-12
    fx = O.fft_vec(x)
    assert abs(np.linalg.norm(fx) ** 2 - n * np.linalg.norm(x) ** 2) / (n * np.linalg.norm(x) ** 2) <= 1e-12


def test_conjugate_fused_forward_transform():  # test_transform.cpp:102-131
    rng = RefRng(61)
    t = rng.tensor(2, 3, 1)
    h1, h2 = O.qfft3_conj(t)
    assert np.array_equal(h1, np.conj(t[0])) and np.array_equal(h2, -t[1])  # p = 1: quaternion conjugation
    # canonical tube (j, 2j, 3j, 4j) -> (-10j, 2j-2k, 2j, 2j+2k)
    t1 = np.zeros((4, 1, 1), np.complex128)
    t2 = np.array([1, 2, 3, 4], np.complex128).reshape(4, 1, 1)
    h1, h2 = O.qfft3_conj((t1, t2))
    want2 = cvec(-10, 2 - 2j, 2, 2 + 2j)
    assert np.all(np.abs(h1.ravel()) <= 1e-13) and np.all(np.abs(h2.ravel() - want2) <= 1e-13)
    # real input: t2 stays exactly zero, t1 = plain fft
    re1 = np.zeros((5, 2, 2), np.complex128)
    re1.real = rng.sym(20).reshape(5, 2, 2)
    h1, h2 = O.qfft3_conj((re1, np.zeros_like(re1)))
    assert np.all(h2 == 0)
    assert np.all(np.abs(h1[:, 1, 0] - O.fft_vec(re1[:, 1, 0])) <= 1e-13)


def test_every_tube_is_sqrt_p_F_conj_q():  # test_transform.cpp:133-152
    rng = RefRng(67)
    t = rng.tensor(3, 2, 7)
    h1, h2 = O.qfft3_conj(t)
    p = 7
    F = np.exp(-2j * np.pi * np.outer(np.arange(p), np.arange(p)) / p)  # sqrt(p) * F_p
    w1 = np.einsum("sr,rij->sij", F, np.conj(t[0]))
    w2 = np.einsum("sr,rij->sij", F, -t[1])
    worst = np.max(np.sqrt(np.abs(h1 - w1) ** 2 + np.abs(h2 - w2) ** 2))
    norm = np.sqrt(np.sum(np.abs(t[0]) ** 2) + np.sum(np.abs(t[1]) ** 2))
    assert worst / norm <= 1e-12


def test_inverse_transform_exact_inverse():  # test_transform.cpp:154-168
    rng = RefRng(71)
    t = rng.tensor(3, 4, 5)
    assert O.rel_frob_error(O.qifft3_conj(O.qfft3_conj(t)), t) <= 1e-12
    assert O.rel_frob_error(O.qfft3_conj(O.qifft3_conj(t)), t) <= 1e-12
    z = (np.zeros((3, 2, 2), np.complex128), np.zeros((3, 2, 2), np.complex128))
    hz = O.qifft3_conj(z)
    assert np.all(hz[0] == 0) and np.all(hz[1] == 0)
    one = (np.array([[[1 + 2j]]]), np.array([[[3 + 4j]]]))
    o1, o2 = O.qifft3_conj(one)
    assert o1[0, 0, 0] == 1 - 2j and o2[0, 0, 0] == -3 - 4j


def test_transform_rejects_p0():
    with pytest.raises(O.OracleError):
        O.qfft3_conj((np.zeros((0, 2, 2), np.complex128), np.zeros((0, 2, 2), np.complex128)))


# ---------------------------------------------------------- test_tproduct.cpp
def test_definitional_product_basics():  # test_tproduct.cpp:60-86
    rng = RefRng(7)
    a = rng.tensor(3, 2, 1)
    b = rng.tensor(2, 4, 1)
    c = O.tprod_naive(a, b)
    # p = 1: plain quaternion matrix product (linalg.hpp:90)
    w1 = a[0][0] @ b[0][0] - a[1][0] @ np.conj(b[1][0])
    w2 = a[0][0] @ b[1][0] + a[1][0] @ np.conj(b[0][0])
    assert np.sqrt(qerr(c[0][0], w1) ** 2 + qerr(c[1][0], w2) ** 2) <= 1e-14
    # right identity
    t = rng.tensor(3, 4, 6)
    eye = (np.zeros((6, 4, 4), np.complex128), np.zeros((6, 4, 4), np.complex128))
    eye[0][0] = np.eye(4)
    assert O.rel_frob_error(O.tprod_naive(t, eye), t) <= 1e-12
    with pytest.raises(O.OracleError):
        O.tprod_naive(a, rng.tensor(3, 2, 1))


def test_fast_equals_naive_reference_cases():  # test_tproduct.cpp:88-116
    rng = RefRng(11)
    a, b = rng.tensor(5, 4, 6), rng.tensor(4, 3, 6)
    assert O.rel_frob_error(O.tprod_fast(a, b), O.tprod_naive(a, b)) <= 1e-11
    a, b = rng.tensor(2, 3, 1), rng.tensor(3, 2, 1)
    assert O.rel_frob_error(O.tprod_fast(a, b), O.tprod_naive(a, b)) <= 1e-13
    for _ in range(60):
        m, n = 1 + rng.next_u64() % 8, 1 + rng.next_u64() % 8
        s, p = 1 + rng.next_u64() % 8, 1 + rng.next_u64() % 12
        a, b = rng.tensor(m, n, p), rng.tensor(n, s, p)
        assert O.rel_frob_error(O.tprod_fast(a, b), O.tprod_naive(a, b)) <= 1e-11


def test_acceptance_criterion_1():  # acceptance.cpp:46-65
    rng = RefRng(20240001)
    worst = 0.0
    for _ in range(100):
        m, n = 1 + rng.next_u64() % 8, 1 + rng.next_u64() % 8
        s, p = 1 + rng.next_u64() % 8, 1 + rng.next_u64() % 12
        a = O.gen_random_tensor(m, n, p, rng.next_u64())
        b = O.gen_random_tensor(n, s, p, rng.next_u64())
        worst = max(worst, O.rel_frob_error(O.tprod_fast(a, b), O.tprod_naive(a, b)))
    assert worst <= 1e-11
    a = O.gen_random_tensor(50, 50, 10, 1001)
    b = O.gen_random_tensor(50, 50, 10, 1002)
    assert O.rel_frob_error(O.tprod_fast(a, b), O.tprod_naive(a, b)) <= 1e-12


def test_slice_reflect_and_flops():  # test_tproduct.cpp:47-58, 186-199
    f = O.flops_estimate(1, 1, 1, 2)
    assert f[2] == 64 and f[0] == 32
    for m, n, s, p in ((1, 1, 1, 2), (3, 4, 5, 7), (20, 20, 20, 64)):
        e = O.flops_estimate(m, n, s, p)
        assert e[2] == e[0] * p
        assert e[3] == 4 * m * p * s * (n * p - 1) + 12 * m * n * s * p * p
    assert O.flops_estimate(1, 1, 1, 1)[1] == 0
    with pytest.raises(O.OracleError):
        O.flops_estimate(0, 1, 1, 1)


def test_generator_determinism():  # acceptance.cpp:306-308
    a = O.gen_random_tensor(4, 5, 3, 7)
    b = O.gen_random_tensor(4, 5, 3, 7)
    assert bits_equal(a[0], b[0]) and bits_equal(a[1], b[1])


# ------------------------------------------------------- golden (reference)
def test_oracle_bitwise_equals_reference_fixtures(small_golden):
    g = small_golden
    for k in range(int(g["ncases"])):
        m, n, s, p = (int(v) for v in g[f"c{k}_shape"])
        a = (g[f"c{k}_a1"], g[f"c{k}_a2"])
        b = (g[f"c{k}_b1"], g[f"c{k}_b2"])
        ga = O.gen_random_tensor(m, n, p, 101 + 2 * k)
        assert bits_equal(ga[0], a[0]) and bits_equal(ga[1], a[1])  # generator == reference generator
        f = O.tprod_fast(a, b)
        assert bits_equal(f[0], g[f"c{k}_fast1"]) and bits_equal(f[1], g[f"c{k}_fast2"]), (m, n, s, p)
        nv = O.tprod_naive(a, b)
        assert bits_equal(nv[0], g[f"c{k}_naive1"]) and bits_equal(nv[1], g[f"c{k}_naive2"]), (m, n, s, p)
        fa = O.qfft3_conj(a)
        assert bits_equal(fa[0], g[f"c{k}_fa1"]) and bits_equal(fa[1], g[f"c{k}_fa2"])
        ia = O.qifft3_conj(a)
        assert bits_equal(ia[0], g[f"c{k}_ia1"]) and bits_equal(ia[1], g[f"c{k}_ia2"])


def test_oracle_config1_matches_reference_fixture(cfg_golden):
    g = cfg_golden
    a = O.gen_random_tensor(32, 32, 16, int(g["cfg1_seeds"][0]))
    b = O.gen_random_tensor(32, 32, 16, int(g["cfg1_seeds"][1]))
    f = O.tprod_fast(a, b)
    assert bits_equal(f[0], g["cfg1_full_fast1"]) and bits_equal(f[1], g["cfg1_full_fast2"])
    assert O.rel_frob_error(f, O.tprod_naive(a, b)) <= 1e-12


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_oracle_bitwise_equals_live_reference():
    rng = np.random.default_rng(5)
    for (m, n, s, p) in [(4, 6, 5, 13), (10, 3, 7, 24), (2, 9, 2, 49), (6, 6, 6, 64), (1, 1, 1, 1)]:
        a = tuple(rng.standard_normal((p, m, n)) + 1j * rng.standard_normal((p, m, n)) for _ in range(2))
        b = tuple(rng.standard_normal((p, n, s)) + 1j * rng.standard_normal((p, n, s)) for _ in range(2))
        f, r = O.tprod_fast(a, b), O.ref_tprod_fast(a, b)
        assert bits_equal(f[0], r[0]) and bits_equal(f[1], r[1])
    assert O.derive_seed(42, 9) == O.ref_derive_seed(42, 9)
    assert O.flops_estimate(20, 20, 20, 64) == O.ref_flops_estimate(20, 20, 20, 64)
