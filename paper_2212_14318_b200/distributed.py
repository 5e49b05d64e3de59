"""Launcher side of the per-rank multi-GPU drivers (one process per GPU).

The drivers themselves are C++ behind the C-ABI (csrc/qt_rank.cu): the
library owns the NCCL communicator, the partition, the exchange schedule and
every transfer.  This module only (1) moves the 128-byte NCCL id from rank 0
to the others over whatever torch.distributed group the launcher set up, and
(2) holds each rank's device buffers.

* RowsTProduct — the north_star split (BASELINE.json): rank r owns a
  contiguous slab of rows of A and C (shard.row_slab); B is broadcast from the
  root by ncclBroadcast inside qt_rank_tprod_rows, then the single-GPU
  product runs on the slab.
* FreqTProduct — frequency-parallel: rank r transforms its rows of A and B,
  owns a contiguous range of frequency slots for stage 2 and its rows of C
  for the inverse transform; the pieces move by NCCL send/recv
  (qt_rank_freq_*), or — after set_peers() with every rank's CUDA IPC handle —
  by K1's own stores into the owners' buffers and K3's own loads from them
  (no messages; the library's device barrier between the phases).  Nothing
  is replicated.
Both are bitwise identical to the single-GPU product (tests/test_gpu_rank.py),
and their schedules are exercised over gloo on CPU
(tests/test_multiproc_gloo.py).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native, shard


class RankComm:
    """This rank's NCCL communicator inside the product library.  `dist_mod`:
    an initialised torch.distributed (any backend) used once to broadcast
    the NCCL id from rank 0; None for a one-rank communicator."""

    def __init__(self, rank: int, world: int, device: int, dist_mod=None):
        self.rank, self.world, self.device = rank, world, device
        L = _native.lib()
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            _native.check(L.qt_comm_unique_id(uid), "ncclGetUniqueId")
        if world > 1:
            box = [bytes(uid.raw) if rank == 0 else None]
            dist_mod.broadcast_object_list(box, src=0)
            uid = ctypes.create_string_buffer(box[0], 128)
        h = ctypes.c_void_p()
        _native.check(L.qt_comm_init(uid, rank, world, device, ctypes.byref(h)), "ncclCommInitRank")
        self.handle = h

    def close(self) -> None:
        if self.handle:
            _native.check(_native.lib().qt_comm_destroy(self.handle), "ncclCommDestroy")
            self.handle = None


def partition(m: int, n: int, p: int, world: int, rank: int):
    """(a0, a1, b0, b1, slot0, slot1) of `rank` (the library's rule, equal to
    shard.row_slab / shard.slot_ranges)."""
    out = (ctypes.c_uint64 * 6)()
    _native.check(_native.lib().qt_rank_partition(m, n, p, world, rank, out), "qt_rank_partition")
    return tuple(int(v) for v in out)


def schedule(m: int, n: int, s: int, p: int, world: int, rank: int, part: str, send: bool):
    """The library's exchange schedule of `rank` for part 'a' / 'b' / 'c': a
    list of (peer, slot, plane, first row, rows) in transfer order."""
    L = _native.lib()
    k = {"a": 0, "b": 1, "c": 2}[part]
    cnt = ctypes.c_uint64()
    _native.check(L.qt_rank_freq_schedule(m, n, s, p, world, rank, k, int(send), None, 0, ctypes.byref(cnt)),
                  "qt_rank_freq_schedule")
    buf = (ctypes.c_int64 * (5 * max(1, cnt.value)))()
    _native.check(L.qt_rank_freq_schedule(m, n, s, p, world, rank, k, int(send), buf, cnt.value, ctypes.byref(cnt)),
                  "qt_rank_freq_schedule")
    return [tuple(buf[5 * i:5 * i + 5]) for i in range(cnt.value)]


class _RankBase:
    def __init__(self, comm: RankComm, m: int, n: int, s: int, p: int, device=None):
        import torch
        self.torch = torch
        self.comm = comm
        self.m, self.n, self.s, self.p = m, n, s, p
        self.rank, self.world = comm.rank, comm.world
        self.dev = torch.device("cuda", comm.device) if device is None else torch.device(device)
        self.L = _native.lib()

    def _planes(self, rows: int, cols: int):
        return self.torch.empty((2, self.p, rows, 2 * cols), dtype=self.torch.float64, device=self.dev)

    def _load(self, dst, src1: np.ndarray, src2: np.ndarray, lo: int, hi: int) -> None:
        for k, src in enumerate((src1, src2)):
            dst[k].copy_(self.torch.from_numpy(np.ascontiguousarray(src[:, lo:hi]).view(np.float64)))

    @staticmethod
    def _stream(stream):
        import torch
        return (torch.cuda.current_stream() if stream is None else stream).cuda_stream

    def result(self):
        """(c1, c2) of this rank's rows as host complex128 (p, rows, s)."""
        out = self.c.cpu().numpy().view(np.complex128)
        return out[0], out[1]


class RowsTProduct(_RankBase):
    """Rows of A and C in slabs, B broadcast from `root` (qt_rank_tprod_rows)."""

    def __init__(self, comm: RankComm, m: int, n: int, s: int, p: int, root: int = 0, device=None):
        super().__init__(comm, m, n, s, p, device)
        self.root = root
        self.a0, self.a1 = shard.row_slab(m, self.world, self.rank)
        self.rows = self.a1 - self.a0
        self.a = self._planes(self.rows, n)
        self.b = self._planes(n, s)
        self.c = self._planes(self.rows, s)

    def load_a(self, a1: np.ndarray, a2: np.ndarray) -> None:
        self._load(self.a, a1, a2, self.a0, self.a1)

    def load_b(self, b1: np.ndarray, b2: np.ndarray) -> None:
        """B (only the root's copy matters: the step broadcasts it)."""
        self._load(self.b, b1, b2, 0, self.n)

    def owned(self):
        """The device buffers this rank fills from the host (its inputs)."""
        return [self.a] + ([self.b] if self.rank == self.root else [])

    def step(self, stream=None) -> None:
        _native.check(self.L.qt_rank_tprod_rows(
            self.comm.handle, self.a[0].data_ptr(), self.a[1].data_ptr(), self.b[0].data_ptr(), self.b[1].data_ptr(),
            self.c[0].data_ptr(), self.c[1].data_ptr(), self.rows, self.n, self.s, self.p, self.root,
            self._stream(stream)), "qt_rank_tprod_rows")


class IpcGroup:
    """rank / world / device of a frequency-parallel plan whose exchange goes
    through peer memory only (no NCCL communicator: qt_rank_freq_create_ipc)."""

    def __init__(self, rank: int, world: int, device: int):
        self.rank, self.world, self.device = rank, world, device
        self.handle = None


class FreqTProduct(_RankBase):
    """Frequency-parallel T-product (qt_rank_freq_*): rows [a0, a1) of A and C,
    rows [b0, b1) of B, stage 2 of the frequency slots [slot0, slot1).  With a
    RankComm the exchange is NCCL send/recv until set_peers() switches it to the
    fused peer-memory exchange; with an IpcGroup it is fused only."""

    def __init__(self, comm, m: int, n: int, s: int, p: int, device=None):
        super().__init__(comm, m, n, s, p, device)
        self.a0, self.a1, self.b0, self.b1, self.slot0, self.slot1 = partition(m, n, p, self.world, self.rank)
        self.rows = self.a1 - self.a0
        self.a = self._planes(self.rows, n)
        self.b = self._planes(self.b1 - self.b0, s)
        self.c = self._planes(self.rows, s)
        h = ctypes.c_void_p()
        if isinstance(comm, IpcGroup):
            _native.check(self.L.qt_rank_freq_create_ipc(comm.rank, comm.world, comm.device, m, n, s, p,
                                                         ctypes.byref(h)), "qt_rank_freq_create_ipc")
        else:
            _native.check(self.L.qt_rank_freq_create(comm.handle, m, n, s, p, ctypes.byref(h)), "qt_rank_freq_create")
        self.plan = h

    def ipc_handle(self) -> bytes:
        """This rank's stage buffer as a 64-byte CUDA IPC handle."""
        buf = ctypes.create_string_buffer(64)
        _native.check(self.L.qt_rank_freq_ipc_handle(self.plan, buf), "qt_rank_freq_ipc_handle")
        return bytes(buf.raw)

    def set_peers(self, handles) -> None:
        """Every rank's ipc_handle() in rank order: switch to the fused exchange."""
        blob = ctypes.create_string_buffer(b"".join(handles), 64 * len(handles))
        _native.check(self.L.qt_rank_freq_set_peers(self.plan, blob), "qt_rank_freq_set_peers")

    def phase(self, k: int, stream=None) -> None:
        """One fused phase without the device barriers (0 routed K1, 1 stage 2, 2 routed K3)."""
        _native.check(self.L.qt_rank_freq_phase(
            self.plan, k, self.a[0].data_ptr(), self.a[1].data_ptr(), self.b[0].data_ptr(), self.b[1].data_ptr(),
            self.c[0].data_ptr(), self.c[1].data_ptr(), self._stream(stream)), "qt_rank_freq_phase")

    def load_a(self, a1: np.ndarray, a2: np.ndarray) -> None:
        self._load(self.a, a1, a2, self.a0, self.a1)

    def load_b(self, b1: np.ndarray, b2: np.ndarray) -> None:
        self._load(self.b, b1, b2, self.b0, self.b1)

    def owned(self):
        return [self.a, self.b]

    def step(self, stream=None) -> None:
        _native.check(self.L.qt_rank_freq_step(
            self.plan, self.a[0].data_ptr(), self.a[1].data_ptr(), self.b[0].data_ptr(), self.b[1].data_ptr(),
            self.c[0].data_ptr(), self.c[1].data_ptr(), self._stream(stream)), "qt_rank_freq_step")

    def nonfinite(self) -> bool:
        """The last step's slots met an inf/NaN (their stage 2 then ran on the
        fp64 kernels, as in the single-GPU product)."""
        v = ctypes.c_int()
        _native.check(self.L.qt_rank_freq_nonfinite(self.plan, ctypes.byref(v)), "qt_rank_freq_nonfinite")
        return bool(v.value)

    def close(self) -> None:
        if self.plan:
            _native.check(self.L.qt_rank_freq_destroy(self.plan), "qt_rank_freq_destroy")
            self.plan = None


def emulate_freq(world: int, a1, a2, b1, b2, c1, c2, m: int, n: int, s: int, p: int, stream=None,
                 fused: bool = False) -> None:
    """`world` frequency-parallel ranks in lockstep on the current device
    (qt_rank_freq_emulate: the pieces moved by device copies along the same
    schedule): whole device tensors in, C out — the one-GPU check of the
    decomposition."""
    import torch
    sh = (torch.cuda.current_stream() if stream is None else stream).cuda_stream
    _native.check(_native.lib().qt_rank_freq_emulate(world, int(fused), a1.data_ptr(), a2.data_ptr(), b1.data_ptr(),
                                                     b2.data_ptr(), c1.data_ptr(), c2.data_ptr(), m, n, s, p, sh),
                  "qt_rank_freq_emulate")
