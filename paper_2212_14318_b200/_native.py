"""ctypes binding of the product library ``libqtensor_b200.so`` (C-ABI in
``include/qtensor_b200.h``).

The library is built in-tree by ``__graft_entry__.build()`` / ``make``.  There
is deliberately no fallback: if the shared object is missing or cannot be
loaded, :func:`lib` raises, and every compute call fails loudly.
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libqtensor_b200.so")

QT_OK, QT_EINVAL, QT_ECUDA, QT_ENOMEM, QT_ENCCL, QT_ENODEV = 0, 1, 2, 3, 4, 5
QT_EBADMAGIC, QT_ETRUNCATED, QT_EDIMOVERFLOW, QT_EIO = 6, 7, 8, 9
QT_DIST_UNIFORM_SYM, QT_DIST_NORMAL, QT_DIST_PURE_UNIT = 0, 1, 2

# Every symbol include/qtensor_b200.h declares: name -> (restype, argtypes)
_u64 = ctypes.c_uint64
_dp = ctypes.c_void_p  # double* (host or device), passed as raw addresses
_vp = ctypes.c_void_p
SIGNATURES = {
    "qt_abi_version": (ctypes.c_int, []),
    "qt_last_error": (ctypes.c_char_p, []),
    "qt_kernel_launches": (_u64, []),
    "qt_prof_enable": (None, [ctypes.c_int]),
    "qt_prof_timeline": (ctypes.c_int, [ctypes.c_char_p, _u64]),
    "qt_prof_read": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64)]),
    "qt_tprod_f64_device": (ctypes.c_int, [_dp] * 6 + [_u64] * 4 + [_vp]),
    "qt_qfft3_conj_f64_device": (ctypes.c_int, [_dp] * 4 + [_u64] * 3 + [_vp]),
    "qt_qifft3_conj_f64_device": (ctypes.c_int, [_dp] * 4 + [_u64] * 3 + [_vp]),
    "qt_fft_routable": (ctypes.c_int, [_u64]),
    "qt_qfft3_conj_f64_device_routed": (ctypes.c_int, [_dp] * 4 + [_u64] * 3 + [_vp]),
    "qt_qifft3_conj_f64_device_routed": (ctypes.c_int, [_dp] * 4 + [_u64] * 3 + [_vp]),
    "qt_qfft3_conj_f64_device_routed_n": (ctypes.c_int, [_dp] * 4 + [ctypes.c_int] + [_u64] * 3 + [_vp]),
    "qt_spectral_product_f64_device": (ctypes.c_int, [_dp] * 6 + [_u64] * 4 + [_vp]),
    "qt_spectral_product_f64_device_ld": (ctypes.c_int, [_dp] * 6 + [_u64] * 8 + [_vp]),
    "qt_spectral_product_f64_device_ld_algo": (ctypes.c_int, [_dp] * 6 + [_u64] * 8 + [ctypes.c_int, _vp]),
    "qt_gemm_algo": (ctypes.c_int, [_u64] * 4),
    "qt_small_fused": (ctypes.c_int, [_u64] * 4),
    "qt_int8_guard_fallbacks": (_u64, []),
    "qt_slot_frequency": (ctypes.c_int, [_u64, _u64]),
    "qt_int8_slots_create": (ctypes.c_int, [_dp, _dp] + [_u64] * 3 + [ctypes.c_int, ctypes.c_int, _vp, _vp,
                                                                      ctypes.POINTER(ctypes.c_void_p)]),
    "qt_int8_slots_multiply": (ctypes.c_int, [ctypes.c_void_p, _dp, _dp, _u64, _dp, _dp, _vp]),
    "qt_int8_slots_destroy": (ctypes.c_int, [ctypes.c_void_p, _vp]),
    "qt_tprod_naive_f64_device": (ctypes.c_int, [_dp] * 6 + [_u64] * 4 + [_vp]),
    "qt_tprod_naive_f64_host": (ctypes.c_int, [_dp] * 6 + [_u64] * 4 + [ctypes.c_int]),
    "qt_tprod_f64_host": (ctypes.c_int, [_dp] * 6 + [_u64] * 4 + [ctypes.c_int]),
    "qt_tprod_f64_host_spectra": (ctypes.c_int, [_dp] * 6 + [_u64] * 4 + [ctypes.c_int] + [_dp] * 6),
    "qt_qfft3_conj_f64_host": (ctypes.c_int, [_dp] * 4 + [_u64] * 3 + [ctypes.c_int]),
    "qt_qifft3_conj_f64_host": (ctypes.c_int, [_dp] * 4 + [_u64] * 3 + [ctypes.c_int]),
    "qt_tprod_f64_multi": (ctypes.c_int, [_dp] * 6 + [_u64] * 4 + [ctypes.POINTER(ctypes.c_int), ctypes.c_int]),
    "qt_comm_unique_id": (ctypes.c_int, [_vp]),
    "qt_comm_init": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "qt_comm_destroy": (ctypes.c_int, [_vp]),
    "qt_rank_partition": (ctypes.c_int, [_u64, _u64, _u64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_u64)]),
    "qt_rank_freq_schedule": (ctypes.c_int, [_u64] * 4 + [ctypes.c_int] * 4 + [ctypes.POINTER(ctypes.c_int64), _u64,
                                                                           ctypes.POINTER(_u64)]),
    "qt_rank_tprod_rows": (ctypes.c_int, [_vp] + [_dp] * 6 + [_u64] * 4 + [ctypes.c_int, _vp]),
    "qt_rank_freq_create": (ctypes.c_int, [_vp] + [_u64] * 4 + [ctypes.POINTER(ctypes.c_void_p)]),
    "qt_rank_freq_step": (ctypes.c_int, [_vp] + [_dp] * 6 + [_vp]),
    "qt_rank_freq_nonfinite": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int)]),
    "qt_rank_freq_destroy": (ctypes.c_int, [_vp]),
    "qt_rank_freq_emulate": (ctypes.c_int, [ctypes.c_int, ctypes.c_int] + [_dp] * 6 + [_u64] * 4 + [_vp]),
    "qt_rank_freq_create_ipc": (ctypes.c_int, [ctypes.c_int] * 3 + [_u64] * 4 + [ctypes.POINTER(ctypes.c_void_p)]),
    "qt_rank_freq_ipc_handle": (ctypes.c_int, [_vp, _vp]),
    "qt_rank_freq_set_peers": (ctypes.c_int, [_vp, _vp]),
    "qt_rank_freq_phase": (ctypes.c_int, [_vp, ctypes.c_int] + [_dp] * 6 + [_vp]),
    "qt_qt3_probe": (ctypes.c_int, [ctypes.c_char_p] + [ctypes.POINTER(ctypes.c_uint64)] * 3),
    "qt_qt3_read_f64_device": (ctypes.c_int, [ctypes.c_char_p, _dp, _dp] + [_u64] * 3 + [_vp]),
    "qt_qt3_write_f64_device": (ctypes.c_int, [ctypes.c_char_p, _dp, _dp] + [_u64] * 3 + [_vp]),
    "qt_gen_tensor_f64": (ctypes.c_int, [ctypes.c_int] + [_u64] * 4 + [ctypes.c_double, _dp, _dp]),
    "qt_derive_seed": (_u64, [_u64, _u64]),
}

_lock = threading.Lock()
_lib = None


class TensorIoError(RuntimeError):
    """QT3 header/payload errors (the reference's TensorIoError, tensor_io.hpp:22-32)."""

    KINDS = {6: "BadMagic", 7: "Truncated", 8: "DimOverflow"}

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.kind = self.KINDS.get(code, "Io")


class QtError(RuntimeError):
    """A non-EINVAL failure reported by the C-ABI (CUDA, NCCL, memory, device)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"qtensor_b200 error {code}: {msg}")
        self.code = code


def lib() -> ctypes.CDLL:
    """Load (once) and return the product library; raises if it is missing."""
    global _lib
    with _lock:
        if _lib is None:
            # QTB_LIB_PATH: another build of this library (A/B timing of two builds on one box)
            path = os.environ.get("QTB_LIB_PATH") or LIB_PATH
            if not os.path.exists(path):
                raise ImportError(
                    f"{path} is missing: build it with `make` or __graft_entry__.build(); "
                    "there is no CPU fallback")
            handle = ctypes.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                if path != LIB_PATH and not hasattr(handle, name):
                    continue  # an older build without this entry point
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
        return _lib


def check(rc: int, who: str) -> None:
    """Map a C-ABI status to the reference's exception kinds."""
    if rc == QT_OK:
        return
    msg = (lib().qt_last_error() or b"").decode(errors="replace")
    if rc == QT_EINVAL:
        raise ValueError(f"{who}: {msg}")  # std::invalid_argument in the reference
    if rc in (QT_EBADMAGIC, QT_ETRUNCATED, QT_EDIMOVERFLOW, QT_EIO):
        raise TensorIoError(rc, f"{who}: {msg}")
    raise QtError(rc, f"{who}: {msg}")
