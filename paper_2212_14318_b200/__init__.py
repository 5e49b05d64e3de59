"""paper_2212_14318_b200 — B200-native drop-in for the reference's fast
quaternion-tensor T-product (``qtensor::tprod_fast``, arXiv 2212.14318).

The compute path is the C-ABI library ``libqtensor_b200.so`` (sm_100a CUDA
kernels); this package is the host-side mirror of the reference interface.
"""
from . import _native
from .configs import CONFIGS, Config, make_inputs
from .tproduct import (CdTensor3, TProdWorkspace, TprodFlops, derive_seed, flops_estimate, gen_random_tensor,
                       gen_tensor, qfft3_conj, qfft3_conj_device, qifft3_conj, qifft3_conj_device, slice_reflect,
                       spectral_product_device, tprod_fast, tprod_fast_device, tprod_fast_multi, tprod_naive)

__all__ = [
    "CdTensor3", "TProdWorkspace", "TprodFlops", "tprod_fast", "tprod_fast_device", "tprod_fast_multi", "tprod_naive",
    "qfft3_conj", "qifft3_conj", "qfft3_conj_device", "qifft3_conj_device", "spectral_product_device",
    "slice_reflect", "flops_estimate", "gen_random_tensor", "gen_tensor", "derive_seed",
    "CONFIGS", "Config", "make_inputs", "_native",
]
