"""Host-side mirror of the reference's T-product interface, backed by the
sm_100a kernels through the C-ABI (``include/qtensor_b200.h``).

Same names, argument meaning and error behaviour as the reference's C++ API
(``/root/reference/proj/include/qtensor/tproduct.hpp:12-56`` and
``transform.hpp:26-64``) so tests read like the reference's own tests:

* :class:`CdTensor3` — quaternion tensor in Cayley-Dickson form Q = t1 + t2 j,
  p frontal m x n slices, slice-major (``transform.hpp:26-54``).  Here ``t1``
  and ``t2`` are complex128 numpy arrays of shape (p, m, n), which is exactly
  the reference's flat ``(r*m + i)*n + j`` order.
* :func:`tprod_fast` (``tproduct.hpp:45-46``), :func:`qfft3_conj`,
  :func:`qifft3_conj` (``transform.hpp:60-64``) run on the GPU; a dimension
  mismatch or p == 0 raises ``ValueError`` where the reference throws
  ``std::invalid_argument`` (``tproduct.cpp:76-77``, ``transform.cpp:152``).
* :func:`slice_reflect`, :func:`flops_estimate`, :class:`TProdWorkspace`,
  :func:`gen_random_tensor`, :func:`derive_seed` mirror the rest of the surface.

There is no CPU path: without the built library or a B200 the calls raise.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native

__all__ = [
    "CdTensor3", "TProdWorkspace", "TprodFlops", "tprod_fast", "tprod_naive", "qfft3_conj", "qifft3_conj",
    "slice_reflect", "flops_estimate", "gen_random_tensor", "gen_tensor", "derive_seed",
    "tprod_fast_device", "qfft3_conj_device", "qifft3_conj_device", "spectral_product_device",
    "tprod_fast_multi",
]


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


class CdTensor3:
    """Third-order quaternion tensor, CD form, slice-major (transform.hpp:26-54)."""

    __slots__ = ("m", "n", "p", "t1", "t2")

    def __init__(self, m: int, n: int, p: int, t1=None, t2=None):
        self.m, self.n, self.p = int(m), int(n), int(p)
        shape = (self.p, self.m, self.n)
        self.t1 = np.zeros(shape, np.complex128) if t1 is None else np.ascontiguousarray(t1, np.complex128).reshape(shape)
        self.t2 = np.zeros(shape, np.complex128) if t2 is None else np.ascontiguousarray(t2, np.complex128).reshape(shape)

    def size(self) -> int:
        return self.m * self.n * self.p

    def idx(self, i: int, j: int, r: int) -> int:
        return (r * self.m + i) * self.n + j

    def qat(self, i: int, j: int, r: int):
        """(w, x, y, z) of entry (i, j, r): t1 = w + x i, t2 = y + z i (algebra.hpp:61-68)."""
        a, b = self.t1[r, i, j], self.t2[r, i, j]
        return (a.real, a.imag, b.real, b.imag)

    def set_qat(self, i: int, j: int, r: int, q) -> None:
        w, x, y, z = q
        self.t1[r, i, j] = complex(w, x)
        self.t2[r, i, j] = complex(y, z)

    def slice(self, r: int):
        return self.t1[r].copy(), self.t2[r].copy()

    def frob_norm(self) -> float:
        return float(np.sqrt(np.sum(np.abs(self.t1) ** 2) + np.sum(np.abs(self.t2) ** 2)))

    def copy(self) -> "CdTensor3":
        return CdTensor3(self.m, self.n, self.p, self.t1.copy(), self.t2.copy())

    def __repr__(self) -> str:
        return f"CdTensor3(m={self.m}, n={self.n}, p={self.p})"


@dataclass
class TProdWorkspace:
    """Reusable state for tprod_fast (tproduct.hpp:31-34).

    The reference keeps host copies of Â, B̂, Ĉ here.  The device pipeline keeps
    its transformed operands in stream-ordered device scratch, so these fields
    stay unspecified (None); reuse is bitwise identical to a fresh call, which
    is the contract test_tproduct.cpp:118-128 pins."""
    ahat: CdTensor3 | None = None
    bhat: CdTensor3 | None = None
    chat: CdTensor3 | None = None


@dataclass(frozen=True)
class TprodFlops:
    fast_mults: int
    fast_transform_flops: int
    naive_mults: int
    naive_adds: int


def slice_reflect(i: int, p: int) -> int:
    """σ(i) = (p - i) mod p, tproduct.hpp:27-29."""
    return (p - i) % p


def flops_estimate(m: int, n: int, s: int, p: int) -> TprodFlops:
    """Operation counts of both routes, tproduct.cpp:113-126 (zero dims raise)."""
    if m == 0 or n == 0 or s == 0 or p == 0:
        raise ValueError("flops_estimate: zero dims")
    lg = float(np.log2(p)) if p > 1 else 0.0
    # std::llround: half away from zero
    x = 2.0 * float(m * n + n * s + m * s) * float(p) * lg
    return TprodFlops(16 * m * n * s * p, int(np.floor(x + 0.5)), 16 * m * n * s * p * p,
                      4 * m * p * s * (n * p - 1) + 12 * m * n * s * p * p)


def _device_index(device) -> int:
    if device is None:
        return 0
    return int(getattr(device, "index", device) or 0)


def tprod_fast(a: CdTensor3, b: CdTensor3, ws: TProdWorkspace | None = None, device=None) -> CdTensor3:
    """C = A *_T B on the GPU (tprod_fast, tproduct.hpp:45-46)."""
    if a.n != b.m or a.p != b.p:
        raise ValueError("tprod_fast: dimension mismatch")
    m, n, s, p = a.m, a.n, b.n, a.p
    c = CdTensor3(m, s, p)
    L = _native.lib()
    rc = L.qt_tprod_f64_host(_ptr(a.t1), _ptr(a.t2), _ptr(b.t1), _ptr(b.t2), _ptr(c.t1), _ptr(c.t2),
                             m, n, s, p, _device_index(device))
    _native.check(rc, "tprod_fast")
    return c


def tprod_naive(a: CdTensor3, b: CdTensor3, device=None) -> CdTensor3:
    """Definitional product fold(bcirc(a) . unfold(b)) on the GPU
    (tprod_naive, tproduct.hpp:23-25): C_k = sum_r A_{(k-r) mod p} (.) B_r."""
    if a.n != b.m or a.p != b.p:
        raise ValueError("tprod_naive: dimension mismatch")
    m, n, s, p = a.m, a.n, b.n, a.p
    c = CdTensor3(m, s, p)
    rc = _native.lib().qt_tprod_naive_f64_host(_ptr(a.t1), _ptr(a.t2), _ptr(b.t1), _ptr(b.t2), _ptr(c.t1),
                                               _ptr(c.t2), m, n, s, p, _device_index(device))
    _native.check(rc, "tprod_naive")
    return c


def tprod_fast_multi(a: CdTensor3, b: CdTensor3, devices) -> CdTensor3:
    """Row-sharded single-process multi-GPU T-product (B broadcast over NCCL)."""
    try:  # load torch's bundled NCCL first: the C library reuses an already-loaded libnccl.so.2
        import torch  # noqa: F401
    except ImportError:
        pass
    if a.n != b.m or a.p != b.p:
        raise ValueError("tprod_fast: dimension mismatch")
    m, n, s, p = a.m, a.n, b.n, a.p
    c = CdTensor3(m, s, p)
    devs = (ctypes.c_int * len(devices))(*devices)
    rc = _native.lib().qt_tprod_f64_multi(_ptr(a.t1), _ptr(a.t2), _ptr(b.t1), _ptr(b.t2), _ptr(c.t1),
                                          _ptr(c.t2), m, n, s, p, devs, len(devices))
    _native.check(rc, "tprod_fast_multi")
    return c


def _transform(q: CdTensor3, inverse: bool, device) -> CdTensor3:
    out = CdTensor3(q.m, q.n, q.p)
    L = _native.lib()
    fn = L.qt_qifft3_conj_f64_host if inverse else L.qt_qfft3_conj_f64_host
    rc = fn(_ptr(q.t1), _ptr(q.t2), _ptr(out.t1), _ptr(out.t2), q.m, q.n, q.p, _device_index(device))
    _native.check(rc, "qifft3_conj" if inverse else "qfft3_conj")
    return out


def qfft3_conj(q: CdTensor3, device=None) -> CdTensor3:
    """out.t1 = fft(conj(t1), 3), out.t2 = -fft(t2, 3) (transform.hpp:56-60)."""
    return _transform(q, False, device)


def qifft3_conj(qhat: CdTensor3, device=None) -> CdTensor3:
    """out.t1 = conj(ifft(t1, 3)), out.t2 = -ifft(t2, 3) (transform.hpp:62-64)."""
    return _transform(qhat, True, device)


# ---------------------------------------------------------------- device API
def _dptr(t) -> int:
    """Device address of a contiguous float64/complex128 torch tensor."""
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("device entry points need contiguous CUDA tensors")
    return t.data_ptr()


def _stream_handle(stream) -> int:
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return int(getattr(stream, "cuda_stream", stream))


def tprod_fast_device(a1, a2, b1, b2, c1, c2, m: int, n: int, s: int, p: int, stream=None) -> None:
    """Device-resident T-product on torch CUDA buffers (enqueued on ``stream``)."""
    rc = _native.lib().qt_tprod_f64_device(_dptr(a1), _dptr(a2), _dptr(b1), _dptr(b2), _dptr(c1), _dptr(c2),
                                           m, n, s, p, _stream_handle(stream))
    _native.check(rc, "tprod_fast")


def qfft3_conj_device(x1, x2, y1, y2, m: int, n: int, p: int, stream=None) -> None:
    rc = _native.lib().qt_qfft3_conj_f64_device(_dptr(x1), _dptr(x2), _dptr(y1), _dptr(y2), m, n, p,
                                                _stream_handle(stream))
    _native.check(rc, "qfft3_conj")


def qifft3_conj_device(x1, x2, y1, y2, m: int, n: int, p: int, stream=None) -> None:
    rc = _native.lib().qt_qifft3_conj_f64_device(_dptr(x1), _dptr(x2), _dptr(y1), _dptr(y2), m, n, p,
                                                 _stream_handle(stream))
    _native.check(rc, "qifft3_conj")


def spectral_product_device(ah1, ah2, bh1, bh2, ch1, ch2, m: int, n: int, s: int, p: int, stream=None) -> None:
    rc = _native.lib().qt_spectral_product_f64_device(_dptr(ah1), _dptr(ah2), _dptr(bh1), _dptr(bh2), _dptr(ch1),
                                                      _dptr(ch2), m, n, s, p, _stream_handle(stream))
    _native.check(rc, "spectral_product")


# ------------------------------------------------------------------ inputs
def derive_seed(base: int, stream: int) -> int:
    """rng.cpp:15-19."""
    return int(_native.lib().qt_derive_seed(base, stream))


def gen_tensor(m: int, n: int, p: int, seed: int, dist: int = _native.QT_DIST_UNIFORM_SYM,
               scale: float = 1.0, out: tuple | None = None) -> CdTensor3:
    """Seeded synthetic tensor (see qt_gen_tensor_f64 in include/qtensor_b200.h)."""
    t = CdTensor3(m, n, p) if out is None else out
    rc = _native.lib().qt_gen_tensor_f64(dist, m, n, p, seed, scale, _ptr(t.t1), _ptr(t.t2))
    _native.check(rc, "gen_random_tensor")
    return t


def gen_random_tensor(m: int, n: int, p: int, seed: int) -> CdTensor3:
    """Bitwise the reference's gen_random_tensor (rng.cpp:21-33)."""
    return gen_tensor(m, n, p, seed, _native.QT_DIST_UNIFORM_SYM)
