"""CPU ORACLE — test infrastructure only.

Python bindings of the two CPU checkers:

* ``liboracle.so`` — this repo's plain-C restatement of the reference hot path
  (``oracle/qt_oracle.c``; each function cites the reference file:line it
  follows);
* ``_ref/libqtref.so`` — the reference itself, compiled from its own sources
  under /root/reference by ``oracle/Makefile`` (``make ref``), namespace
  renamed to ``qtref``; present on the GPU box only as the prebuilt .so.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may import this package, and only as the checker or the timed
CPU baseline — never as the product path.

Tensors are (t1, t2) pairs of complex128 numpy arrays of shape (p, m, n)
(slice-major, transform.hpp:35-37).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(_HERE, "liboracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libqtref.so")

_u64 = ctypes.c_uint64
_p = ctypes.c_void_p
_orc = None
_ref = None


def _load_oracle():
    global _orc
    if _orc is None:
        L = ctypes.CDLL(ORACLE_SO)
        L.orc_derive_seed.restype = _u64
        L.orc_derive_seed.argtypes = [_u64, _u64]
        for nm, args in {
            "orc_gen_random_tensor": [_u64, _u64, _u64, _u64, _p, _p],
            "orc_gen_tensor": [ctypes.c_int, _u64, _u64, _u64, _u64, ctypes.c_double, _p, _p],
            "orc_rng_sym_stream": [_u64, _u64, _p],
            "orc_rng_u64_stream": [_u64, _u64, _p],
            "orc_dft_vec_naive": [_p, _u64, _p],
            "orc_fft_vec": [_p, _u64, _p],
            "orc_ifft_vec": [_p, _u64, _p],
            "orc_qfft3_conj": [_p, _p, _p, _p, _u64, _u64, _u64],
            "orc_qifft3_conj": [_p, _p, _p, _p, _u64, _u64, _u64],
            "orc_tprod_fast": [_p] * 6 + [_u64] * 4,
            "orc_tprod_naive": [_p] * 6 + [_u64] * 4,
            "orc_flops_estimate": [_u64] * 4 + [_p],
        }.items():
            f = getattr(L, nm)
            f.restype = ctypes.c_int
            f.argtypes = args
        L.orc_rel_frob_error.restype = ctypes.c_double
        L.orc_rel_frob_error.argtypes = [_p] * 4 + [_u64]
        _orc = L
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _load_ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref, needs /root/reference)")
        L = ctypes.CDLL(REF_SO)
        for nm, args in {
            "ref_tprod_fast": [_p] * 6 + [_u64] * 6,
            "ref_tprod_naive": [_p] * 6 + [_u64] * 6,
            "ref_qfft3_conj": [_p] * 4 + [_u64] * 3,
            "ref_qifft3_conj": [_p] * 4 + [_u64] * 3,
            "ref_fft_vec": [_p, _u64, _p],
            "ref_gen_random_tensor": [_u64] * 4 + [_p, _p],
        }.items():
            f = getattr(L, nm)
            f.restype = ctypes.c_int
            f.argtypes = args
        L.ref_write_tensor.restype = ctypes.c_int
        L.ref_write_tensor.argtypes = [ctypes.c_char_p, _p, _p, _u64, _u64, _u64]
        L.ref_read_tensor.restype = ctypes.c_int
        L.ref_read_tensor.argtypes = [ctypes.c_char_p, _p, _p, _p]
        L.ref_derive_seed.restype = _u64
        L.ref_derive_seed.argtypes = [_u64, _u64]
        L.ref_flops.restype = _u64
        L.ref_flops.argtypes = [_u64] * 4 + [_p]
        _ref = L
    return _ref


def _a(x):
    x = np.ascontiguousarray(x, dtype=np.complex128)
    return x, x.ctypes.data


class OracleError(ValueError):
    """The oracle (or the reference) rejected the arguments (std::invalid_argument)."""


def _chk(rc, who):
    if rc == 1:
        raise OracleError(f"{who}: invalid argument")
    if rc != 0:
        raise RuntimeError(f"{who}: rc={rc}")


# ------------------------------------------------------------ restatement
def derive_seed(base: int, stream: int) -> int:
    return int(_load_oracle().orc_derive_seed(base, stream))


def gen_random_tensor(m, n, p, seed):
    t1 = np.empty((p, m, n), np.complex128)
    t2 = np.empty((p, m, n), np.complex128)
    _chk(_load_oracle().orc_gen_random_tensor(m, n, p, seed, t1.ctypes.data, t2.ctypes.data), "gen_random_tensor")
    return t1, t2


def gen_tensor(dist: int, m, n, p, seed, scale: float = 1.0):
    """The BASELINE input distributions (0 uniform = gen_random_tensor,
    1 normal, 2 pure-quaternion RGB), restated for the reference arm of
    bench.py; bitwise equal to the product library's qt_gen_tensor_f64."""
    t1 = np.empty((p, m, n), np.complex128)
    t2 = np.empty((p, m, n), np.complex128)
    _chk(_load_oracle().orc_gen_tensor(int(dist), m, n, p, seed, ctypes.c_double(scale), t1.ctypes.data,
                                       t2.ctypes.data), "gen_tensor")
    return t1, t2


def rng_sym(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, np.float64)
    _chk(_load_oracle().orc_rng_sym_stream(seed, count, out.ctypes.data), "rng_sym")
    return out


def rng_u64(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, np.uint64)
    _chk(_load_oracle().orc_rng_u64_stream(seed, count, out.ctypes.data), "rng_u64")
    return out


def _vec(fn, x):
    x, px = _a(x)
    y = np.empty_like(x)
    _chk(fn(px, x.size, y.ctypes.data), fn.__name__)
    return y


def dft_vec_naive(x):
    return _vec(_load_oracle().orc_dft_vec_naive, x)


def fft_vec(x):
    return _vec(_load_oracle().orc_fft_vec, x)


def ifft_vec(x):
    return _vec(_load_oracle().orc_ifft_vec, x)


def _transform(fn, q):
    x1, p1 = _a(q[0])
    x2, p2 = _a(q[1])
    p, m, n = x1.shape
    y1 = np.empty_like(x1)
    y2 = np.empty_like(x2)
    _chk(fn(p1, p2, y1.ctypes.data, y2.ctypes.data, m, n, p), fn.__name__)
    return y1, y2


def qfft3_conj(q):
    return _transform(_load_oracle().orc_qfft3_conj, q)


def qifft3_conj(q):
    return _transform(_load_oracle().orc_qifft3_conj, q)


def _tprod(fn, a, b, who):
    a1, pa1 = _a(a[0])
    a2, pa2 = _a(a[1])
    b1, pb1 = _a(b[0])
    b2, pb2 = _a(b[1])
    p, m, n = a1.shape
    bp, bm, s = b1.shape
    if n != bm or p != bp:
        raise OracleError(f"{who}: dimension mismatch")
    c1 = np.empty((p, m, s), np.complex128)
    c2 = np.empty((p, m, s), np.complex128)
    _chk(fn(pa1, pa2, pb1, pb2, c1.ctypes.data, c2.ctypes.data, m, n, s, p), who)
    return c1, c2


def tprod_fast(a, b):
    """Restated tprod_fast (tproduct.cpp:75-106)."""
    return _tprod(_load_oracle().orc_tprod_fast, a, b, "tprod_fast")


def tprod_naive(a, b):
    """Restated definitional product fold(bcirc(a) . unfold(b)) (tproduct.cpp:49-53)."""
    return _tprod(_load_oracle().orc_tprod_naive, a, b, "tprod_naive")


def rel_frob_error(got, want) -> float:
    """rel_frob_error (bench.cpp:30-37)."""
    g1, pg1 = _a(got[0])
    g2, pg2 = _a(got[1])
    w1, pw1 = _a(want[0])
    w2, pw2 = _a(want[1])
    assert g1.shape == w1.shape
    return float(_load_oracle().orc_rel_frob_error(pg1, pg2, pw1, pw2, g1.size))


def flops_estimate(m, n, s, p):
    out = np.zeros(4, np.uint64)
    _chk(_load_oracle().orc_flops_estimate(m, n, s, p, out.ctypes.data), "flops_estimate")
    return [int(v) for v in out]


# --------------------------------------------------- the reference itself
def _ref_tprod(fn, a, b, who):
    a1, pa1 = _a(a[0])
    a2, pa2 = _a(a[1])
    b1, pb1 = _a(b[0])
    b2, pb2 = _a(b[1])
    p, m, n = a1.shape
    bp, bm, s = b1.shape
    c1 = np.empty((p, m, s), np.complex128)
    c2 = np.empty((p, m, s), np.complex128)
    _chk(fn(pa1, pa2, pb1, pb2, c1.ctypes.data, c2.ctypes.data, m, n, bm, s, p, bp), who)
    return c1, c2


def ref_tprod_fast(a, b):
    """The UNMODIFIED reference tprod_fast (oracle/_ref)."""
    return _ref_tprod(_load_ref().ref_tprod_fast, a, b, "ref_tprod_fast")


def ref_tprod_naive(a, b):
    return _ref_tprod(_load_ref().ref_tprod_naive, a, b, "ref_tprod_naive")


def ref_qfft3_conj(q):
    return _transform(_load_ref().ref_qfft3_conj, q)


def ref_qifft3_conj(q):
    return _transform(_load_ref().ref_qifft3_conj, q)


def ref_fft_vec(x):
    return _vec(_load_ref().ref_fft_vec, x)


def ref_gen_random_tensor(m, n, p, seed):
    t1 = np.empty((p, m, n), np.complex128)
    t2 = np.empty((p, m, n), np.complex128)
    _chk(_load_ref().ref_gen_random_tensor(m, n, p, seed, t1.ctypes.data, t2.ctypes.data), "ref_gen")
    return t1, t2


def ref_derive_seed(base, stream):
    return int(_load_ref().ref_derive_seed(base, stream))


def ref_flops_estimate(m, n, s, p):
    out = np.zeros(4, np.uint64)
    _chk(int(_load_ref().ref_flops(m, n, s, p, out.ctypes.data)), "ref_flops")
    return [int(v) for v in out]


def ref_write_tensor(path: str, t):
    """The reference's write_tensor (tensor_io.cpp:85-92) on (t1, t2)."""
    t1, p1 = _a(t[0])
    t2, p2 = _a(t[1])
    p, m, n = t1.shape
    rc = _load_ref().ref_write_tensor(path.encode(), p1, p2, m, n, p)
    if rc:
        raise RuntimeError(f"ref_write_tensor rc={rc}")


def ref_read_tensor(path: str):
    """The reference's read_tensor (tensor_io.cpp:94-103): (t1, t2) or an
    int error code 6/7/8 (TensorIoErrorKind BadMagic/Truncated/DimOverflow), 9."""
    dims = np.zeros(3, np.uint64)
    rc = _load_ref().ref_read_tensor(path.encode(), None, None, dims.ctypes.data)
    if rc:
        return rc
    m, n, p = (int(v) for v in dims)
    t1 = np.empty((p, m, n), np.complex128)
    t2 = np.empty((p, m, n), np.complex128)
    rc = _load_ref().ref_read_tensor(path.encode(), t1.ctypes.data, t2.ctypes.data, dims.ctypes.data)
    return (t1, t2) if rc == 0 else rc


def qt3_bytes(t1: np.ndarray, t2: np.ndarray) -> bytes:
    """QT3 serialisation restated (tensor_io.cpp:37-50): magic, m, n, p (LE u64),
    then per entry w, x, y, z (LE f64), slice-major."""
    p, m, n = t1.shape
    rec = np.empty((t1.size, 4), "<f8")
    rec[:, 0] = t1.reshape(-1).real
    rec[:, 1] = t1.reshape(-1).imag
    rec[:, 2] = t2.reshape(-1).real
    rec[:, 3] = t2.reshape(-1).imag
    return b"QT3\x00" + np.array([m, n, p], "<u8").tobytes() + rec.tobytes()
