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
