"""Partition rules of the multi-GPU T-product (one process per GPU).

Row i of C = A *_T B depends only on row i of A and all of B (every slice
product and every tube transform is row-local), so the rows of A
and C are split into contiguous slabs of ceil(m / world) rows (row split: B
broadcast); stage 2 is independent per frequency pair, so the frequency-
parallel split gives each rank a contiguous range of frequency slots.

These are restatements of the C++ drivers' rules (csrc/qt_rank.cu,
csrc/qt_multi.cu) for the CPU tests; tests/test_multiproc_gloo.py checks the
two agree (qt_rank_partition).
"""
from __future__ import annotations

from typing import Callable

import numpy as np


def row_slab(m: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) rows of rank `rank`: contiguous slabs of ceil(m/world) rows."""
    slab = -(-m // world)
    lo = min(m, rank * slab)
    hi = min(m, lo + slab)
    return lo, hi


def slot_freq(p: int, slot: int) -> int:
    """Frequency of stage-2 slot `slot` (qt_slot_frequency): slots 2j, 2j+1
    hold the pair (j+1, p-j-1); the self-paired 0 (and p/2 for even p) come
    last (csrc/qt_ozaki.cu slot_freq)."""
    npairs = (p - 1) // 2
    if slot < 2 * npairs:
        return p - (slot // 2 + 1) if slot & 1 else slot // 2 + 1
    return 0 if slot == 2 * npairs else p // 2


def slot_ranges(p: int, world: int) -> list[tuple[int, int]]:
    """Contiguous slot ranges [s0, s1), one per rank, for the frequency-
    parallel decomposition.  Every slot costs the same stage-2 GEMM (a pair is
    two slots, a self-paired frequency one), so the boundaries sit at the
    nearest slot to k p / world that does not split a pair (an odd slot below
    2 ((p - 1) / 2)): range sizes differ by at most 2 slots."""
    pair_end = 2 * ((p - 1) // 2)
    bounds = [0]
    for k in range(1, world):
        ideal = k * p / world
        b = int(round(ideal))
        if b & 1 and b < pair_end:
            b = b - 1 if ideal < b else b + 1
        bounds.append(min(p, max(bounds[-1], b)))
    bounds.append(p)
    return list(zip(bounds[:-1], bounds[1:]))


def take_rows(t1: np.ndarray, t2: np.ndarray, lo: int, hi: int):
    """Rows [lo, hi) of a slice-major (p, m, n) tensor, as a contiguous slab."""
    return np.ascontiguousarray(t1[:, lo:hi, :]), np.ascontiguousarray(t2[:, lo:hi, :])


def sharded_tprod(a_slab, b, compute: Callable, broadcast: Callable, rank: int):
    """One rank's share of the row-sharded T-product.

    a_slab    : this rank's rows of A (already resident on the rank)
    b         : B on rank 0 (a preallocated receive buffer elsewhere)
    broadcast : broadcast(buffers, src=0) over the process group (NCCL on
                GPUs; gloo in the CPU tests)
    compute   : compute(a_slab, b) -> C slab (the GPU pipeline, or the oracle
                in the CPU tests)
    """
    broadcast(b, 0)
    return compute(a_slab, b)
