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
    single-GPU int8 product (row and column scalings and the contraction
    balancing depend on the slot's own data only), so the stitched C is
    bitwise identical to it.  Inputs holding inf/NaN, and pairs the int8
    accuracy guard does not certify, are recomputed by the fp64 DMMA kernels
    on the compact slot tensors (qt_int8_slots_multiply), as in the
    single-GPU product; nonfinite() reports the former.
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
        """True if this rank's slots met an inf/NaN (stage 2 of its slots then
        ran on the fp64 DMMA kernels)."""
        return bool(self.flag.item())

    def result(self):
        """(c1, c2) of this rank's rows as host complex128 (p, rows, s)."""
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
