"""Row sharding of the T-product over ranks (one process per GPU).

Row i of C = A *_T B depends only on row i of A and all of B (every slice
product and every tube transform is row-local), so the rows of A
and C are split into contiguous slabs of ceil(m / world) rows and B is
replicated by broadcasts of its column chunks, each from the rank that owns
(uploaded) it — the only exchange on the path.  The
slab computation is the single-GPU pipeline unchanged, so the stitched result
is bitwise identical to the one-GPU result for every world size.

The same slab rule is used by the C++ single-process driver
(qt_tprod_f64_multi, csrc/qt_multi.cu).
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


def column_chunks(s: int, nchunks: int, world: int, tile: int = 16) -> list[tuple[int, int, int]]:
    """B's column chunks as (c0, c1, owner): ~nchunks chunks of a multiple of
    `tile` columns, owned round-robin.  The owner of chunk j holds (uploads)
    those columns of B and is the root of their broadcast, so with G ranks each
    rank moves ~1/G of B over its PCIe link and its NVLink egress instead of
    rank 0 moving all of it."""
    q = -(-s // max(1, nchunks))
    q = min(s, -(-q // tile) * tile) if s else 0
    if q == 0:
        return []
    return [(c0, min(s, c0 + q), j % max(1, world)) for j, c0 in enumerate(range(0, s, q))]


def split_range(lo: int, hi: int, parts: int, tile: int = 1) -> list[tuple[int, int]]:
    """[lo, hi) in `parts` contiguous pieces of ceil(len/parts) rounded up to a
    multiple of `tile` (trailing pieces may be empty)."""
    n = hi - lo
    q = -(-n // max(1, parts))
    q = -(-q // tile) * tile if q else 0
    return [(min(hi, lo + k * q), min(hi, lo + (k + 1) * q)) for k in range(parts)]


def grid_shape(world: int, m: int, s: int) -> tuple[int, int]:
    """(gr, gc) with gr * gc = world for the 2-D block decomposition of C.
    Every rank of row group i needs the residues/transform of A's row block i
    and every rank of column group j those of B's column block j, so the
    per-rank replicated work is ~ m/gr + s/gc: minimise it (ties: more row
    groups).  world = 2 gives (2, 1), i.e. plain row sharding."""
    best = None
    for gr in range(1, world + 1):
        if world % gr:
            continue
        gc = world // gr
        cost = m / gr + s / gc
        if best is None or cost < best[0] - 1e-12 or (abs(cost - best[0]) <= 1e-12 and gr > best[1]):
            best = (cost, gr, gc)
    return best[1], best[2]


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
