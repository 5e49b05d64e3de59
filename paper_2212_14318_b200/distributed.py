"""One rank's share of the row-sharded T-product, with B broadcast in column
chunks that overlap the compute (one process per GPU, torch.distributed/NCCL
for the plumbing).

Row i of C depends only on row i of A, and column j of C only on column j of
B.  Rank r owns rows shard.row_slab(m, world, r) of A and C; B
lives as NJ column chunks owned round-robin by the ranks (shard.column_chunks)
and is broadcast chunk by chunk from each owner (async NCCL collectives on
the process group's stream).  The compute stream
transforms the A slab once, then for every chunk j waits only for chunk j's
broadcast, transforms it (K1) and runs the paired-frequency GEMM (K2) straight
into columns [c0_j, c1_j) of the C slab (qt_spectral_product_f64_device_ld);
one inverse transform (K3) of the slab finishes the step.  So the transfer of
chunk j+1 overlaps the K1/K2 of chunk j, and only chunk 0's broadcast is
exposed.  Every element is computed with the same kernels and the same
arithmetic as the single-GPU path: the stitched C is bitwise identical for
every world size and chunk count (tests/test_gpu_parity.py).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native, shard


class RowShardedTProduct:
    def __init__(self, m: int, n: int, s: int, p: int, rank: int = 0, world: int = 1, device=None,
                 nchunks: int = 8):
        import torch
        self.torch = torch
        self.m, self.n, self.s, self.p = m, n, s, p
        self.rank, self.world = rank, world
        self.dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.lo, self.hi = shard.row_slab(m, world, rank)
        self.rows = self.hi - self.lo
        plan = shard.column_chunks(s, nchunks, world)  # multiples of the GEMM column tile
        self.chunks = [(c0, c1) for c0, c1, _ in plan]
        self.owner = [o for _, _, o in plan]
        f64 = dict(dtype=torch.float64, device=self.dev)
        self.a = torch.empty((2, p, self.rows, 2 * n), **f64)
        self.ah = torch.empty_like(self.a)
        self.bc = [torch.empty((2, p, n, 2 * (c1 - c0)), **f64) for c0, c1 in self.chunks]
        self.bh = [torch.empty_like(t) for t in self.bc]
        self.c = torch.empty((2, p, self.rows, 2 * s), **f64)
        self.L = _native.lib()
        # one stage-2 algorithm for every rank and chunk: the full product's
        # (QT_GEMM_DMMA or QT_GEMM_INT8_EXACT), so the stitched C is bitwise
        # identical to a single-GPU call
        self.algo = self.L.qt_gemm_algo(m, n, s, p)

    # ---------------------------------------------------------------- inputs
    def load_a(self, a1: np.ndarray, a2: np.ndarray) -> None:
        """Rows of this rank from full host planes (p, m, n) complex128."""
        for k, src in enumerate((a1, a2)):
            slab = np.ascontiguousarray(src[:, self.lo:self.hi]).view(np.float64)
            self.a[k].copy_(self.torch.from_numpy(slab))

    def owned(self, j: int) -> bool:
        return self.owner[j] == self.rank

    def load_b(self, b1: np.ndarray, b2: np.ndarray, owned_only: bool = True) -> None:
        """The chunks of B (p, n, s host planes) this rank owns into their
        buffers (all chunks with owned_only=False: one rank run without peers)."""
        for j, (t, (c0, c1)) in enumerate(zip(self.bc, self.chunks)):
            if owned_only and not self.owned(j):
                continue
            for k, src in enumerate((b1, b2)):
                t[k].copy_(self.torch.from_numpy(np.ascontiguousarray(src[:, :, c0:c1]).view(np.float64)))

    # ----------------------------------------------------------------- step
    def step(self, broadcast=None, stream=None) -> None:
        """One T-product step.  `broadcast(tensor, src)` must enqueue an async
        broadcast from rank `src` (the chunk's owner) and return an object with
        .wait() (a torch.distributed Work); None on a single rank."""
        torch = self.torch
        st = torch.cuda.current_stream() if stream is None else stream
        sh = st.cuda_stream
        L, n, s, p, rows = self.L, self.n, self.s, self.p, self.rows
        works = [broadcast(t, o) for t, o in zip(self.bc, self.owner)] if broadcast is not None else None
        if rows:
            _native.check(L.qt_qfft3_conj_f64_device(self.a[0].data_ptr(), self.a[1].data_ptr(),
                                                     self.ah[0].data_ptr(), self.ah[1].data_ptr(), rows, n, p, sh),
                          "qfft3_conj(A slab)")
        plan = None
        if rows and self.algo == 1:
            # exact int8 stage 2: the residues of this rank's Â slab are built
            # once per step and reused by every B̂ chunk
            h = ctypes.c_void_p()
            _native.check(L.qt_int8_plan_create(self.ah[0].data_ptr(), self.ah[1].data_ptr(), rows, n, p, sh,
                                                ctypes.byref(h)), "int8 plan")
            plan = h
        for j, (c0, c1) in enumerate(self.chunks):
            if works is not None:
                works[j].wait()  # compute stream waits for chunk j only
            if not rows:
                continue
            cols = c1 - c0
            _native.check(L.qt_qfft3_conj_f64_device(self.bc[j][0].data_ptr(), self.bc[j][1].data_ptr(),
                                                     self.bh[j][0].data_ptr(), self.bh[j][1].data_ptr(), n, cols, p,
                                                     sh), "qfft3_conj(B chunk)")
            off = 16 * c0  # bytes: column c0 of every row of the C slab
            if plan is not None:
                _native.check(L.qt_int8_plan_multiply(
                    plan, self.bh[j][0].data_ptr(), self.bh[j][1].data_ptr(), self.c[0].data_ptr() + off,
                    self.c[1].data_ptr() + off, cols, cols, s, n * cols, rows * s, sh), "int8 plan multiply")
            else:
                _native.check(L.qt_spectral_product_f64_device_ld_algo(
                    self.ah[0].data_ptr(), self.ah[1].data_ptr(), self.bh[j][0].data_ptr(), self.bh[j][1].data_ptr(),
                    self.c[0].data_ptr() + off, self.c[1].data_ptr() + off, rows, n, cols, p,
                    cols, s, n * cols, rows * s, self.algo, sh), "spectral_product(chunk)")
        if plan is not None:
            _native.check(L.qt_int8_plan_destroy(plan, sh), "int8 plan destroy")
        if rows:
            _native.check(L.qt_qifft3_conj_f64_device(self.c[0].data_ptr(), self.c[1].data_ptr(),
                                                      self.c[0].data_ptr(), self.c[1].data_ptr(), rows, s, p, sh),
                          "qifft3_conj(C slab)")

    def result(self):
        """(c1, c2) of this rank's rows as host complex128 (p, rows, s)."""
        out = self.c.cpu().numpy().view(np.complex128)
        return out[0], out[1]


class Grid2DTProduct:
    """One rank's share of the 2-D block-decomposed T-product (gr x gc ranks).

    Rank (i, j) = divmod(rank, gc) computes block (rows of row block i, columns
    of column block j) of C.  Row i of C needs only row i of A and column j
    only column j of B, so a block needs A's row block i and
    B's column block j.  Those arrive inside the step: A's row block is split
    into gc pieces, piece k owned (resident, uploaded) by rank (i, k) and
    broadcast over its row group; B's column block into gr pieces, piece k
    owned by rank (k, j) and broadcast over its column group.  Per rank: K1 of
    each arriving A piece into the Â block, then the stage-2 residues of Â
    (int8 path: one plan), then per arriving B piece K1 + stage 2 into its
    columns of the C block, then K3.  Against row sharding (gc = 1) the
    replicated work per rank — the transform and residues of ALL of B — drops
    to those of one column block: config 5 at 8 ranks, (gr, gc) = (4, 2).
    Every element goes through the same kernels and arithmetic as the
    single-GPU product (the stage-2 algorithm is the full shape's), so the
    stitched C is bitwise identical for every grid.
    """

    def __init__(self, m: int, n: int, s: int, p: int, rank: int = 0, world: int = 1, device=None, grid=None,
                 stage_buffer=None):
        import torch
        self.torch = torch
        self.m, self.n, self.s, self.p = m, n, s, p
        self.rank, self.world = rank, world
        self.gr, self.gc = grid if grid is not None else shard.grid_shape(world, m, s)
        assert self.gr * self.gc == world
        self.i, self.j = divmod(rank, self.gc)
        self.dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.r0, self.r1 = shard.row_slab(m, self.gr, self.i)
        self.c0, self.c1 = shard.split_range(0, s, self.gc, tile=16)[self.j]
        self.rows, self.cols = self.r1 - self.r0, self.c1 - self.c0
        # pieces: (lo, hi, owner rank)
        self.apieces = [(lo, hi, self.i * self.gc + k)
                        for k, (lo, hi) in enumerate(shard.split_range(self.r0, self.r1, self.gc))]
        self.bpieces = [(lo, hi, k * self.gc + self.j)
                        for k, (lo, hi) in enumerate(shard.split_range(self.c0, self.c1, self.gr, tile=16))]
        f64 = dict(dtype=torch.float64, device=self.dev)
        self.a = [torch.empty((2, p, hi - lo, 2 * n), **f64) for lo, hi, _ in self.apieces]
        self.ah_p = [torch.empty_like(t) for t in self.a]
        self.b = [torch.empty((2, p, n, 2 * (hi - lo)), **f64) for lo, hi, _ in self.bpieces]
        # Â block and B̂ pieces: carved out of `stage_buffer` (e.g. symmetric
        # memory the group's owners store into) or allocated here
        sizes = self.stage_sizes(m, n, s, p, world, (self.gr, self.gc))[rank]
        if stage_buffer is None:
            stage_buffer = torch.empty(sum(sizes), **f64)
        assert stage_buffer.dtype == torch.float64 and stage_buffer.numel() >= sum(sizes)
        self.stage_buffer = stage_buffer
        self.ah = stage_buffer[:sizes[0]].view(2, p, self.rows, 2 * n)
        self.bh, off = [], sizes[0]
        for lo, hi, _ in self.bpieces:
            e = 2 * p * n * 2 * (hi - lo)
            self.bh.append(stage_buffer[off:off + e].view(2, p, n, 2 * (hi - lo)))
            off += e
        self.c = torch.empty((2, p, self.rows, 2 * self.cols), **f64)
        self.L = _native.lib()
        self.algo = self.L.qt_gemm_algo(m, n, s, p)
        self.tables = None

    @staticmethod
    def stage_sizes(m: int, n: int, s: int, p: int, world: int, grid):
        """Per rank: float64 elements of (its Â block, all its B̂ pieces)."""
        gr, gc = grid
        out = []
        for r in range(world):
            i, j = divmod(r, gc)
            r0, r1 = shard.row_slab(m, gr, i)
            c0, c1 = shard.split_range(0, s, gc, tile=16)[j]
            out.append((2 * p * (r1 - r0) * 2 * n, 2 * p * n * 2 * (c1 - c0)))
        return out

    # ------------------------------------------------ broadcast fused into K1
    # With every rank's stage buffer addressable (peer_bases, as seen from this
    # GPU), an owner transforms its piece ONCE and K1's stores put every
    # frequency row of it straight into the Â block (B̂ piece) of each rank of
    # its row (column) group — qt_qfft3_conj_f64_device_routed_n, one table per
    # destination — instead of broadcasting the raw piece for every rank of the
    # group to transform again.
    def set_peers(self, peer_bases) -> None:
        torch, p, n = self.torch, self.p, self.n
        sizes = self.stage_sizes(self.m, n, self.s, p, self.world, (self.gr, self.gc))
        self.tables = {}
        for k, (lo, hi, owner) in enumerate(self.apieces):
            if owner != self.rank or hi == lo:
                continue
            dsts = [self.i * self.gc + jj for jj in range(self.gc)]
            tab = [[peer_bases[d] + 16 * (((pl * p + r) * self.rows + (lo - self.r0)) * n)
                    for d in dsts for r in range(p)] for pl in (0, 1)]
            self.tables[("a", k)] = (torch.tensor(tab, dtype=torch.int64, device=self.dev), len(dsts))
        for k, (lo, hi, owner) in enumerate(self.bpieces):
            if owner != self.rank or hi == lo:
                continue
            dsts = [ii * self.gc + self.j for ii in range(self.gr)]
            before = sum(2 * p * n * 2 * (h - l) for l, h, _ in self.bpieces[:k])
            cols = hi - lo
            tab = [[peer_bases[d] + 8 * (sizes[d][0] + before) + 16 * ((pl * p + r) * n * cols)
                    for d in dsts for r in range(p)] for pl in (0, 1)]
            self.tables[("b", k)] = (torch.tensor(tab, dtype=torch.int64, device=self.dev), len(dsts))

    def k1_fused(self, stream=None) -> None:
        """K1 of this rank's own pieces, stored into every rank of their groups."""
        st = self.torch.cuda.current_stream() if stream is None else stream
        for (kind, k), (tab, nd) in self.tables.items():
            x = self.a[k] if kind == "a" else self.b[k]
            lo, hi, _ = (self.apieces if kind == "a" else self.bpieces)[k]
            rows, width = (hi - lo, self.n) if kind == "a" else (self.n, hi - lo)
            _native.check(self.L.qt_qfft3_conj_f64_device_routed_n(
                x[0].data_ptr(), x[1].data_ptr(), tab[0].data_ptr(), tab[1].data_ptr(), nd, rows, width, self.p,
                st.cuda_stream), f"qfft3_conj routed ({kind} piece)")

    def step_fused(self, barrier, stream=None) -> None:
        """One step with the piece broadcasts fused into the owners' K1:
        K1 of own pieces → barrier → stage 2 of every B̂ piece → barrier → K3
        (the second barrier: no rank still reads the Â/B̂ the next K1 rewrites)."""
        self.k1_fused(stream)
        barrier()
        self._stage2(stream)
        barrier()
        self._k3(stream)

    # ---------------------------------------------------------------- inputs
    def owns_a(self, k: int) -> bool:
        return self.apieces[k][2] == self.rank

    def owns_b(self, k: int) -> bool:
        return self.bpieces[k][2] == self.rank

    def load_a(self, a1: np.ndarray, a2: np.ndarray, owned_only: bool = True) -> None:
        for k, (lo, hi, _) in enumerate(self.apieces):
            if (owned_only and not self.owns_a(k)) or hi == lo:
                continue
            for t, src in enumerate((a1, a2)):
                self.a[k][t].copy_(self.torch.from_numpy(np.ascontiguousarray(src[:, lo:hi]).view(np.float64)))

    def load_b(self, b1: np.ndarray, b2: np.ndarray, owned_only: bool = True) -> None:
        for k, (lo, hi, _) in enumerate(self.bpieces):
            if (owned_only and not self.owns_b(k)) or hi == lo:
                continue
            for t, src in enumerate((b1, b2)):
                self.b[k][t].copy_(self.torch.from_numpy(np.ascontiguousarray(src[:, :, lo:hi]).view(np.float64)))

    # ----------------------------------------------------------------- step
    def step(self, bcast_row=None, bcast_col=None, stream=None) -> None:
        """One step.  bcast_row(tensor, src) / bcast_col(tensor, src) enqueue
        an async broadcast from global rank `src` over this rank's row /
        column group and return a Work (None: no peers in that group)."""
        torch = self.torch
        st = torch.cuda.current_stream() if stream is None else stream
        sh = st.cuda_stream
        L, n, p = self.L, self.n, self.p
        wa = [bcast_row(t, o) if hi > lo else None for t, (lo, hi, o) in zip(self.a, self.apieces)] \
            if bcast_row is not None else None
        wb = [bcast_col(t, o) if hi > lo else None for t, (lo, hi, o) in zip(self.b, self.bpieces)] \
            if bcast_col is not None else None
        for k, (lo, hi, _) in enumerate(self.apieces):
            if wa is not None and wa[k] is not None:
                wa[k].wait()
            if hi == lo:
                continue
            one = len(self.apieces) == 1
            dst = self.ah if one else self.ah_p[k]
            _native.check(L.qt_qfft3_conj_f64_device(self.a[k][0].data_ptr(), self.a[k][1].data_ptr(),
                                                     dst[0].data_ptr(), dst[1].data_ptr(), hi - lo, n, p, sh),
                          "qfft3_conj(A piece)")
            if not one:
                self.ah[:, :, lo - self.r0:hi - self.r0].copy_(self.ah_p[k])
        self._stage2(stream, wb=wb, transform_b=True)
        self._k3(stream)

    def _stage2(self, stream=None, wb=None, transform_b=False) -> None:
        """Stage 2 of every B̂ piece into its columns of the C block (after
        transforming the arrived raw piece when transform_b)."""
        torch = self.torch
        st = torch.cuda.current_stream() if stream is None else stream
        sh = st.cuda_stream
        L, n, p = self.L, self.n, self.p
        plan = None
        if self.rows and self.algo == 1:
            h = ctypes.c_void_p()
            _native.check(L.qt_int8_plan_create(self.ah[0].data_ptr(), self.ah[1].data_ptr(), self.rows, n, p, sh,
                                                ctypes.byref(h)), "int8 plan")
            plan = h
        for k, (lo, hi, _) in enumerate(self.bpieces):
            if wb is not None and wb[k] is not None:
                wb[k].wait()
            if hi == lo or not self.rows:
                continue
            cols = hi - lo
            if transform_b:
                _native.check(L.qt_qfft3_conj_f64_device(self.b[k][0].data_ptr(), self.b[k][1].data_ptr(),
                                                         self.bh[k][0].data_ptr(), self.bh[k][1].data_ptr(), n, cols,
                                                         p, sh), "qfft3_conj(B piece)")
            off = 16 * (lo - self.c0)
            if plan is not None:
                _native.check(L.qt_int8_plan_multiply(
                    plan, self.bh[k][0].data_ptr(), self.bh[k][1].data_ptr(), self.c[0].data_ptr() + off,
                    self.c[1].data_ptr() + off, cols, cols, self.cols, n * cols, self.rows * self.cols, sh),
                    "int8 plan multiply")
            else:
                _native.check(L.qt_spectral_product_f64_device_ld_algo(
                    self.ah[0].data_ptr(), self.ah[1].data_ptr(), self.bh[k][0].data_ptr(), self.bh[k][1].data_ptr(),
                    self.c[0].data_ptr() + off, self.c[1].data_ptr() + off, self.rows, n, cols, p,
                    cols, self.cols, n * cols, self.rows * self.cols, self.algo, sh), "spectral_product(piece)")
        if plan is not None:
            _native.check(L.qt_int8_plan_destroy(plan, sh), "int8 plan destroy")

    def _k3(self, stream=None) -> None:
        st = self.torch.cuda.current_stream() if stream is None else stream
        if self.rows and self.cols:
            _native.check(self.L.qt_qifft3_conj_f64_device(self.c[0].data_ptr(), self.c[1].data_ptr(),
                                                           self.c[0].data_ptr(), self.c[1].data_ptr(), self.rows,
                                                           self.cols, self.p, st.cuda_stream), "qifft3_conj(C block)")

    def result(self):
        """(c1, c2) of this rank's block as host complex128 (p, rows, cols)."""
        out = self.c.cpu().numpy().view(np.complex128)
        return out[0], out[1]


class FreqParallelTProduct:
    """One rank's share of the frequency-parallel T-product (int8 stage 2).

    The three stages partition along different axes, with one exchange
    between neighbours and no replicated work:
      K1  tube FFTs are independent per (row, column) tube: rank r transforms
          its rows [a0, a1) of A (shard.row_slab(m)) and rows [b0, b1) of B
          (shard.row_slab(n));
      K2  stage 2 is independent per frequency pair (k, p - k): rank r owns
          the slot range shard.slot_ranges(p)[r] and runs the exact int8 GEMM
          on compact operands holding just those slots, for all of m, n, s
          (qt_int8_slots_*: B' residues once, then Â);
      K3  the inverse tube FFTs of rank r's rows [a0, a1) of C.
    Between them, each (slot, rows) piece goes point to point from the rank
    that transformed it to the rank that needs it: Â[k] rows [a0, a1) and
    B̂[k] rows [b0, b1) to the owner of k's slot, Ĉ[k] rows of rank i back to
    rank i — every piece a contiguous block of both the sender's and the
    receiver's buffer, so the exchange is a group of NCCL send/recv pairs
    straight from and into the stage buffers.  Per rank that is 1/G of every
    kernel's work plus (G-1)/G of its own Â, B̂ and Ĉ rows over NVLink, where
    the 2-D block decomposition replicates the transforms and residues of a
    whole row block of A and column block of B.

    Every slot is evaluated with the same kernels and arithmetic as the
    single-GPU int8 product (row and column scalings depend on the slot's
    own data only), so the stitched C is bitwise identical to it.  Inputs
    holding inf/NaN are detected (nonfinite()) and rejected by result(): the
    fp64 DMMA decomposition (Grid2DTProduct) handles those.
    """

    def __init__(self, m: int, n: int, s: int, p: int, rank: int = 0, world: int = 1, device=None,
                 stage_buffer=None):
        import torch
        self.torch = torch
        self.m, self.n, self.s, self.p = m, n, s, p
        self.rank, self.world = rank, world
        self.dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.arows = [shard.row_slab(m, world, r) for r in range(world)]
        self.brows = [shard.row_slab(n, world, r) for r in range(world)]
        self.ranges = shard.slot_ranges(p, world)
        self.a0, self.a1 = self.arows[rank]
        self.b0, self.b1 = self.brows[rank]
        self.s0, self.s1 = self.ranges[rank]
        self.rows, self.ns = self.a1 - self.a0, self.s1 - self.s0
        self.freq = [shard.slot_freq(p, t) for t in range(p)]
        f64 = dict(dtype=torch.float64, device=self.dev)
        br = self.b1 - self.b0
        self.a = torch.empty((2, p, self.rows, 2 * n), **f64)
        self.ah = torch.empty_like(self.a)
        self.b = torch.empty((2, p, br, 2 * s), **f64)
        self.bh = torch.empty_like(self.b)
        # the compact slot tensors Â/B̂/Ĉ of this rank's slots: carved out of
        # `stage_buffer` (float64, >= stage_doubles(...) elements — e.g. a
        # symmetric-memory buffer its peers can address) or allocated here
        sizes = self.stage_sizes(m, n, s, p, world)[rank]
        if stage_buffer is None:
            stage_buffer = torch.empty(sum(sizes), **f64)
        assert stage_buffer.dtype == torch.float64 and stage_buffer.numel() >= sum(sizes)
        self.stage_buffer = stage_buffer
        o1, o2 = sizes[0], sizes[0] + sizes[1]
        self.ac = stage_buffer[:o1].view(2, self.ns, m, 2 * n)
        self.bc = stage_buffer[o1:o2].view(2, self.ns, n, 2 * s)
        self.cc = stage_buffer[o2:o2 + sizes[2]].view(2, self.ns, m, 2 * s)
        self.tables = None  # routed-exchange row tables (set_peers)
        self.c = torch.empty((2, p, self.rows, 2 * s), **f64)
        self.flag = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.L = _native.lib() if self.dev.type == "cuda" else None

    @staticmethod
    def stage_sizes(m: int, n: int, s: int, p: int, world: int):
        """Per rank: float64 elements of its (Â, B̂, Ĉ) compact slot tensors,
        laid out in that order in its stage buffer."""
        out = []
        for t0, t1 in shard.slot_ranges(p, world):
            ns = t1 - t0
            out.append((2 * ns * m * 2 * n, 2 * ns * n * 2 * s, 2 * ns * m * 2 * s))
        return out

    @staticmethod
    def routable(p: int) -> bool:
        """The tube transforms of length p can route their rows (one pass)."""
        return bool(_native.lib().qt_fft_routable(p))

    @staticmethod
    def eligible(m: int, n: int, s: int, p: int) -> bool:
        """The full product would run stage 2 on the int8 path (so the
        decomposition keeps the single-GPU arithmetic), and the exchange stays
        a modest number of messages (2p per stage buffer and rank)."""
        return _native.lib().qt_gemm_algo(m, n, s, p) == 1 and p <= 1024

    # ---------------------------------------------------------------- inputs
    def load_a(self, a1: np.ndarray, a2: np.ndarray) -> None:
        for k, src in enumerate((a1, a2)):
            self.a[k].copy_(self.torch.from_numpy(np.ascontiguousarray(src[:, self.a0:self.a1]).view(np.float64)))

    def load_b(self, b1: np.ndarray, b2: np.ndarray) -> None:
        for k, src in enumerate((b1, b2)):
            self.b[k].copy_(self.torch.from_numpy(np.ascontiguousarray(src[:, self.b0:self.b1]).view(np.float64)))

    # ----------------------------------------------------- exchange schedule
    # Each list is [(view, peer)] in one fixed order (peer, slot, plane) that
    # the sending and the receiving side enumerate identically, so NCCL's
    # in-order matching of a send/recv pair lines every piece up.
    def sends_a(self):
        if not self.rows:
            return []
        return [(self.ah[pl, self.freq[t]], j) for j, (t0, t1) in enumerate(self.ranges)
                for t in range(t0, t1) for pl in (0, 1)]

    def recvs_a(self):
        return [(self.ac[pl, t - self.s0, r0:r1], i) for i, (r0, r1) in enumerate(self.arows) if r1 > r0
                for t in range(self.s0, self.s1) for pl in (0, 1)]

    def sends_b(self):
        if self.b1 == self.b0:
            return []
        return [(self.bh[pl, self.freq[t]], j) for j, (t0, t1) in enumerate(self.ranges)
                for t in range(t0, t1) for pl in (0, 1)]

    def recvs_b(self):
        return [(self.bc[pl, t - self.s0, r0:r1], i) for i, (r0, r1) in enumerate(self.brows) if r1 > r0
                for t in range(self.s0, self.s1) for pl in (0, 1)]

    def sends_c(self):
        return [(self.cc[pl, t - self.s0, r0:r1], i) for i, (r0, r1) in enumerate(self.arows) if r1 > r0
                for t in range(self.s0, self.s1) for pl in (0, 1)]

    def recvs_c(self):
        if not self.rows:
            return []
        return [(self.c[pl, self.freq[t]], j) for j, (t0, t1) in enumerate(self.ranges)
                for t in range(t0, t1) for pl in (0, 1)]

    # ---------------------------------------------------------------- stages
    def _stream(self, stream):
        return (self.torch.cuda.current_stream() if stream is None else stream).cuda_stream

    def k1(self, stream=None) -> None:
        """Forward tube FFTs of this rank's rows of A and of B."""
        sh, L = self._stream(stream), self.L
        if self.b1 > self.b0:
            _native.check(L.qt_qfft3_conj_f64_device(self.b[0].data_ptr(), self.b[1].data_ptr(), self.bh[0].data_ptr(),
                                                     self.bh[1].data_ptr(), self.b1 - self.b0, self.s, self.p, sh),
                          "qfft3_conj(B rows)")
        if self.rows:
            _native.check(L.qt_qfft3_conj_f64_device(self.a[0].data_ptr(), self.a[1].data_ptr(), self.ah[0].data_ptr(),
                                                     self.ah[1].data_ptr(), self.rows, self.n, self.p, sh),
                          "qfft3_conj(A rows)")

    def k2_prepare(self, stream=None):
        """B' residues of this rank's slots (needs the B̂ exchange only)."""
        if not self.ns:
            return None
        h = ctypes.c_void_p()
        _native.check(self.L.qt_int8_slots_create(self.bc[0].data_ptr(), self.bc[1].data_ptr(), self.n, self.s, self.p,
                                                  self.s0, self.ns, self.flag.data_ptr(), self._stream(stream),
                                                  ctypes.byref(h)), "int8 slots (B')")
        return h

    def k2_multiply(self, h, stream=None) -> None:
        """Ĉ of this rank's slots for all m rows (needs the Â exchange)."""
        if h is None:
            return
        sh = self._stream(stream)
        _native.check(self.L.qt_int8_slots_multiply(h, self.ac[0].data_ptr(), self.ac[1].data_ptr(), self.m,
                                                    self.cc[0].data_ptr(), self.cc[1].data_ptr(), sh),
                      "int8 slots multiply")
        _native.check(self.L.qt_int8_slots_destroy(h, sh), "int8 slots destroy")

    def k3(self, stream=None) -> None:
        if self.rows:
            _native.check(self.L.qt_qifft3_conj_f64_device(self.c[0].data_ptr(), self.c[1].data_ptr(),
                                                           self.c[0].data_ptr(), self.c[1].data_ptr(), self.rows,
                                                           self.s, self.p, self._stream(stream)), "qifft3_conj(C rows)")

    # ------------------------------------------ exchange fused into K1 / K3
    # With every rank's stage buffer addressable (peer_bases: device address of
    # rank j's stage buffer as seen from this GPU — NVLink P2P through
    # symmetric memory, or plain addresses on one device), the exchange needs
    # no messages: K1 stores frequency k of its rows straight into the slot
    # owner's Â/B̂ tensors, and K3 loads frequency k of its rows of Ĉ straight
    # from the owner's — one pointer per frequency and plane
    # (qt_q{i}fft3_conj_f64_device_routed).  The pieces land exactly where the
    # point-to-point exchange puts them, so results are bitwise the same.
    def set_peers(self, peer_bases) -> None:
        torch = self.torch
        assert len(peer_bases) == self.world
        sizes = self.stage_sizes(self.m, self.n, self.s, self.p, self.world)
        slot_of = [0] * self.p
        for t, k in enumerate(self.freq):
            slot_of[k] = t
        owner = [j for j, (t0, t1) in enumerate(self.ranges) for _ in range(t0, t1)]
        m, n, s = self.m, self.n, self.s

        def table(part, rows_total, width, r0):
            # part 0/1/2 = Â/B̂/Ĉ of the owner; element (pl, slot - s0, r0, 0)
            out = [[0] * self.p for _ in range(2)]
            for k in range(self.p):
                t = slot_of[k]
                j = owner[t]
                ns_j = self.ranges[j][1] - self.ranges[j][0]
                base = peer_bases[j] + 8 * sum(sizes[j][:part])
                for pl in (0, 1):
                    out[pl][k] = base + 16 * (((pl * ns_j + (t - self.ranges[j][0])) * rows_total + r0) * width)
            return torch.tensor(out, dtype=torch.int64, device=self.dev)

        self.tables = {"a": table(0, m, n, self.a0), "b": table(1, n, s, self.b0), "c": table(2, m, s, self.a0)}

    def k1_routed(self, stream=None) -> None:
        """K1 with the Â/B̂ exchange fused into its stores."""
        sh, L, T = self._stream(stream), self.L, self.tables
        if self.b1 > self.b0:
            _native.check(L.qt_qfft3_conj_f64_device_routed(self.b[0].data_ptr(), self.b[1].data_ptr(),
                                                            T["b"][0].data_ptr(), T["b"][1].data_ptr(),
                                                            self.b1 - self.b0, self.s, self.p, sh),
                          "qfft3_conj routed (B rows)")
        if self.rows:
            _native.check(L.qt_qfft3_conj_f64_device_routed(self.a[0].data_ptr(), self.a[1].data_ptr(),
                                                            T["a"][0].data_ptr(), T["a"][1].data_ptr(), self.rows,
                                                            self.n, self.p, sh), "qfft3_conj routed (A rows)")

    def k3_routed(self, stream=None) -> None:
        """K3 with the Ĉ exchange fused into its loads."""
        if self.rows:
            T = self.tables
            _native.check(self.L.qt_qifft3_conj_f64_device_routed(T["c"][0].data_ptr(), T["c"][1].data_ptr(),
                                                                  self.c[0].data_ptr(), self.c[1].data_ptr(),
                                                                  self.rows, self.s, self.p,
                                                                  self._stream(stream)), "qifft3_conj routed (C rows)")

    def step_routed(self, barrier, stream=None) -> None:
        """One step with the exchange fused into K1/K3.  `barrier()` is a
        stream-ordered barrier over the ranks: after it, every rank's earlier
        kernels (and so their peer stores) are complete.  Two per step: after
        K1 (the Â/B̂ pieces are in place) and after stage 2 (every Ĉ is
        complete, and no rank still reads Â/B̂ the next step's K1 overwrites);
        the next step's first barrier also orders this step's K3 loads before
        any rank's next stage 2 rewrites its Ĉ."""
        self.flag.zero_()
        self.k1_routed(stream)
        barrier()
        self.k2_multiply(self.k2_prepare(stream), stream)
        barrier()
        self.k3_routed(stream)

    def step(self, exchange=None, stream=None) -> None:
        """One step.  `exchange(sends, recvs)` starts the point-to-point
        transfers and returns a list of Works to wait on (make_exchange);
        None runs a single rank (its own pieces are copied locally)."""
        ex = exchange if exchange is not None else make_exchange(self.rank, None)
        self.flag.zero_()
        self.k1(stream)
        wb = ex(self.sends_b(), self.recvs_b())
        # (the Â transfers are started before waiting for B̂, so they overlap
        # the B' residues)
        wa = ex(self.sends_a(), self.recvs_a())
        for w in wb:
            w.wait()
        h = self.k2_prepare(stream)
        for w in wa:
            w.wait()
        self.k2_multiply(h, stream)
        for w in ex(self.sends_c(), self.recvs_c()):
            w.wait()
        self.k3(stream)

    def nonfinite(self) -> bool:
        """True if this rank's slots met an inf/NaN (its Ĉ was not written)."""
        return bool(self.flag.item())

    def result(self):
        """(c1, c2) of this rank's rows as host complex128 (p, rows, s)."""
        if self.nonfinite():
            raise FloatingPointError("frequency-parallel int8 product: non-finite input values; "
                                     "use Grid2DTProduct (fp64 DMMA stage 2) for this product")
        out = self.c.cpu().numpy().view(np.complex128)
        return out[0], out[1]


def make_exchange(rank: int, dist_mod, group=None):
    """exchange(sends, recvs) over torch.distributed point-to-point ops (NCCL:
    one group of send/recv pairs on the process group's stream; gloo on CPU),
    with the rank's own pieces copied locally; returns the Works to wait on.
    dist_mod None: a single rank, local copies only."""

    def ex(sends, recvs):
        own_src = [v for v, peer in sends if peer == rank]
        own_dst = [v for v, peer in recvs if peer == rank]
        assert len(own_src) == len(own_dst)
        for src, dst in zip(own_src, own_dst):
            dst.copy_(src)
        if dist_mod is None:
            assert len(own_src) == len(sends) and len(own_dst) == len(recvs)
            return []
        ops = [dist_mod.P2POp(dist_mod.isend, v, peer, group) for v, peer in sends if peer != rank]
        ops += [dist_mod.P2POp(dist_mod.irecv, v, peer, group) for v, peer in recvs if peer != rank]
        return dist_mod.batch_isend_irecv(ops) if ops else []

    return ex


def make_peer_stage(m: int, n: int, s: int, p: int, rank: int, world: int, device, dist_mod, group=None):
    """Symmetric-memory stage buffer for FreqParallelTProduct plus the peers'
    base addresses and a device-side barrier: (buffer, peer_bases, barrier).
    Raises if symmetric memory is unavailable (callers fall back to the
    point-to-point exchange)."""
    import torch
    import torch.distributed._symmetric_memory as symm_mem
    sizes = FreqParallelTProduct.stage_sizes(m, n, s, p, world)
    numel = max(sum(x) for x in sizes)
    buf = symm_mem.empty(numel, dtype=torch.float64, device=device)
    grp = group if group is not None else dist_mod.group.WORLD
    hdl = symm_mem.rendezvous(buf, grp)
    bases = [int(x) for x in hdl.buffer_ptrs]

    def barrier():
        hdl.barrier(channel=0)

    return buf, bases, barrier


def emulate_freq_parallel_routed(ranks) -> None:
    """emulate_freq_parallel with the exchange fused into K1/K3: the G
    instances share one device, each one's row tables point into the others'
    stage buffers, and lockstep order stands in for the barriers."""
    bases = [x.stage_buffer.data_ptr() for x in ranks]
    for x in ranks:
        if x.tables is None:
            x.set_peers(bases)
    for x in ranks:
        x.flag.zero_()
        x.k1_routed()
    for x in ranks:
        x.k2_multiply(x.k2_prepare())
    for x in ranks:
        x.k3_routed()


def emulate_grid_fused(ranks) -> None:
    """One step of G Grid2DTProduct instances (rank r = ranks[r]) with the
    piece broadcasts fused into the owners' K1, in lockstep on one device: the
    row tables point into the other instances' stage buffers, and lockstep
    order stands in for the barriers."""
    bases = [x.stage_buffer.data_ptr() for x in ranks]
    for x in ranks:
        if x.tables is None:
            x.set_peers(bases)
    for x in ranks:
        x.k1_fused()
    for x in ranks:
        x._stage2()
    for x in ranks:
        x._k3()


def make_peer_grid_stage(m: int, n: int, s: int, p: int, rank: int, world: int, grid, device, dist_mod,
                         group=None):
    """Symmetric-memory stage buffer for Grid2DTProduct, the peers' base
    addresses and a device barrier (as make_peer_stage)."""
    import torch
    import torch.distributed._symmetric_memory as symm_mem
    numel = max(sum(x) for x in Grid2DTProduct.stage_sizes(m, n, s, p, world, grid))
    buf = symm_mem.empty(numel, dtype=torch.float64, device=device)
    hdl = symm_mem.rendezvous(buf, group if group is not None else dist_mod.group.WORLD)
    bases = [int(x) for x in hdl.buffer_ptrs]

    def barrier():
        hdl.barrier(channel=0)

    return buf, bases, barrier


def emulate_freq_parallel(ranks) -> None:
    """Run one step of G FreqParallelTProduct instances (rank r = ranks[r]) on
    one device in lockstep, moving every exchanged piece by a device copy:
    the single-GPU check of the decomposition (the kernels' results do not
    depend on who runs them)."""

    def route(sends_of, recvs_of):
        inbox = {}
        for r, x in enumerate(ranks):
            for v, peer in sends_of(x):
                inbox.setdefault((r, peer), []).append(v)
        for r, x in enumerate(ranks):
            got = {}
            for v, peer in recvs_of(x):
                i = got.get(peer, 0)
                v.copy_(inbox[(peer, r)][i])
                got[peer] = i + 1
            for peer, cnt in got.items():
                assert cnt == len(inbox[(peer, r)])

    for x in ranks:
        x.flag.zero_()
        x.k1()
    route(lambda x: x.sends_b(), lambda x: x.recvs_b())
    route(lambda x: x.sends_a(), lambda x: x.recvs_a())
    for x in ranks:
        x.k2_multiply(x.k2_prepare())
    route(lambda x: x.sends_c(), lambda x: x.recvs_c())
    for x in ranks:
        x.k3()
