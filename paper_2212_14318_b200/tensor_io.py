"""QT3 tensor files <-> device CD planes, mirroring the
reference's tensor_io (/root/reference/proj/include/qtensor/tensor_io.hpp:14-38):
``read_tensor`` / ``write_tensor`` on host CdTensor3 objects, plus device
variants that stream a file straight into (or out of) the two HBM planes the
T-product consumes.  Header errors raise ``TensorIoError`` with ``.kind`` in
{"BadMagic", "Truncated", "DimOverflow"} like the reference's
TensorIoErrorKind; open/read/write failures raise ``TensorIoError`` kind "Io".
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _native
from ._native import TensorIoError  # noqa: F401  (re-export)
from .tproduct import CdTensor3, _dptr, _stream_handle

__all__ = ["probe", "read_tensor", "write_tensor", "read_tensor_device", "write_tensor_device", "TensorIoError"]


def probe(path: str | os.PathLike) -> tuple[int, int, int]:
    """(m, n, p) from a QT3 header, validated like parse_tensor (no GPU needed)."""
    m, n, p = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    rc = _native.lib().qt_qt3_probe(os.fsencode(path), ctypes.byref(m), ctypes.byref(n), ctypes.byref(p))
    _native.check(rc, "read_tensor")
    return m.value, n.value, p.value


def read_tensor_device(path, device=None, stream=None):
    """Stream a QT3 file into two device planes: returns (t1, t2, m, n, p) with
    t1/t2 float64 CUDA tensors of shape (p, m, 2n) (interleaved re/im)."""
    import torch
    m, n, p = probe(path)
    dev = torch.device("cuda", 0 if device is None else int(getattr(device, "index", device) or 0))
    t1 = torch.empty((p, m, 2 * n), dtype=torch.float64, device=dev)
    t2 = torch.empty_like(t1)
    rc = _native.lib().qt_qt3_read_f64_device(os.fsencode(path), _dptr(t1), _dptr(t2), m, n, p,
                                              _stream_handle(stream))
    _native.check(rc, "read_tensor")
    return t1, t2, m, n, p


def write_tensor_device(path, t1, t2, m: int, n: int, p: int, stream=None) -> None:
    """Write two device planes as a QT3 file (bit-exact)."""
    rc = _native.lib().qt_qt3_write_f64_device(os.fsencode(path), _dptr(t1), _dptr(t2), m, n, p,
                                               _stream_handle(stream))
    _native.check(rc, "write_tensor")


def read_tensor(path, device=None) -> CdTensor3:
    """read_tensor (tensor_io.hpp:38) through the GPU de-interleave."""
    t1, t2, m, n, p = read_tensor_device(path, device)
    h1 = t1.cpu().numpy().view(np.complex128)
    h2 = t2.cpu().numpy().view(np.complex128)
    return CdTensor3(m, n, p, h1, h2)


def write_tensor(path, t: CdTensor3, device=None) -> None:
    """write_tensor (tensor_io.hpp:37) through the GPU interleave."""
    import torch
    dev = torch.device("cuda", 0 if device is None else int(getattr(device, "index", device) or 0))
    d1 = torch.from_numpy(np.ascontiguousarray(t.t1).view(np.float64)).to(dev)
    d2 = torch.from_numpy(np.ascontiguousarray(t.t2).view(np.float64)).to(dev)
    write_tensor_device(path, d1, d2, t.m, t.n, t.p)
