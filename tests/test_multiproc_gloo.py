"""CPU, world_size 2 over gloo: the N>1 host path of bench.py / shard.py.

Each rank holds its row slab of A, rank 0 broadcasts B, each rank computes its
C slab (the oracle stands in for the GPU pipeline on CPU), rank 0 gathers and
the stitched C must equal the single-process result bitwise."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, m, n, s, p, out_path):
    import sys
    sys.path.insert(0, ROOT)
    import oracle as O
    from paper_2212_14318_b200 import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = O.gen_random_tensor(m, n, p, 11)          # every rank can regenerate A; it keeps only its slab
    lo, hi = shard.row_slab(m, world, rank)
    a_slab = shard.take_rows(a[0], a[1], lo, hi)
    if rank == 0:
        b = O.gen_random_tensor(n, s, p, 12)
    else:
        b = (np.zeros((p, n, s), np.complex128), np.zeros((p, n, s), np.complex128))
    bt = [torch.from_numpy(b[0].view(np.float64)), torch.from_numpy(b[1].view(np.float64))]

    def broadcast(_b, src):
        for t in bt:
            dist.broadcast(t, src=src)

    c = shard.sharded_tprod(a_slab, b, lambda x, y: O.tprod_fast(x, y), broadcast, rank)
    # gather slabs (padded to the max slab size) on rank 0
    slab = -(-m // world)
    buf = np.zeros((2, p, slab, s), np.complex128)
    buf[0, :, :hi - lo] = c[0]
    buf[1, :, :hi - lo] = c[1]
    t = torch.from_numpy(buf.view(np.float64))
    gathered = [torch.zeros_like(t) for _ in range(world)] if rank == 0 else None
    dist.gather(t, gathered, dst=0)
    if rank == 0:
        c1 = np.zeros((p, m, s), np.complex128)
        c2 = np.zeros((p, m, s), np.complex128)
        for r, g in enumerate(gathered):
            lo_r, hi_r = shard.row_slab(m, world, r)
            gg = g.numpy().view(np.complex128)
            c1[:, lo_r:hi_r] = gg[0, :, :hi_r - lo_r]
            c2[:, lo_r:hi_r] = gg[1, :, :hi_r - lo_r]
        np.savez(out_path, c1=c1, c2=c2)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("m,n,s,p", [(9, 5, 6, 8), (4, 3, 5, 7), (1, 2, 3, 4)])
def test_row_sharded_world2_equals_single(tmp_path, m, n, s, p):
    import oracle as O
    out = str(tmp_path / "c.npz")
    mp.spawn(_worker, args=(2, _free_port(), m, n, s, p, out), nprocs=2, join=True)
    got = np.load(out)
    a = O.gen_random_tensor(m, n, p, 11)
    b = O.gen_random_tensor(n, s, p, 12)
    want = O.tprod_fast(a, b)
    assert np.array_equal(got["c1"].view(np.uint64), want[0].view(np.uint64))
    assert np.array_equal(got["c2"].view(np.uint64), want[1].view(np.uint64))


def _worker_chunks(rank, world, port, m, n, s, p, nchunks, out_path):
    """B in column chunks owned round-robin (shard.column_chunks): each rank
    fills only the chunks it owns, every chunk is broadcast from its owner,
    then each rank computes its C slab — the N > 1 bench pipeline's schedule."""
    import sys
    sys.path.insert(0, ROOT)
    import oracle as O
    from paper_2212_14318_b200 import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = O.gen_random_tensor(m, n, p, 21)
    lo, hi = shard.row_slab(m, world, rank)
    a_slab = shard.take_rows(a[0], a[1], lo, hi)
    b_full = O.gen_random_tensor(n, s, p, 22)
    plan = shard.column_chunks(s, nchunks, world, tile=1)
    assert len(plan) >= 1 and plan[0][0] == 0 and plan[-1][1] == s
    bufs = []
    for (c0, c1, owner) in plan:
        t1 = np.zeros((p, n, c1 - c0), np.complex128)
        t2 = np.zeros((p, n, c1 - c0), np.complex128)
        if owner == rank:  # only the owner holds (uploads) this chunk
            t1[:] = b_full[0][:, :, c0:c1]
            t2[:] = b_full[1][:, :, c0:c1]
        bufs.append((t1, t2, owner))
    works = []
    for (t1, t2, owner) in bufs:
        for t in (t1, t2):
            works.append(dist.broadcast(torch.from_numpy(t.view(np.float64)), src=owner, async_op=True))
    for w in works:
        w.wait()
    b1 = np.concatenate([t1 for t1, _, _ in bufs], axis=2)
    b2 = np.concatenate([t2 for _, t2, _ in bufs], axis=2)
    assert np.array_equal(b1.view(np.uint64), b_full[0].view(np.uint64))
    assert np.array_equal(b2.view(np.uint64), b_full[1].view(np.uint64))
    c = O.tprod_fast(a_slab, (b1, b2))
    slab = -(-m // world)
    buf = np.zeros((2, p, slab, s), np.complex128)
    buf[0, :, :hi - lo] = c[0]
    buf[1, :, :hi - lo] = c[1]
    t = torch.from_numpy(buf.view(np.float64))
    gathered = [torch.zeros_like(t) for _ in range(world)] if rank == 0 else None
    dist.gather(t, gathered, dst=0)
    if rank == 0:
        c1 = np.zeros((p, m, s), np.complex128)
        c2 = np.zeros((p, m, s), np.complex128)
        for r, g in enumerate(gathered):
            lo_r, hi_r = shard.row_slab(m, world, r)
            gg = g.numpy().view(np.complex128)
            c1[:, lo_r:hi_r] = gg[0, :, :hi_r - lo_r]
            c2[:, lo_r:hi_r] = gg[1, :, :hi_r - lo_r]
        np.savez(out_path, c1=c1, c2=c2)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("m,n,s,p,nchunks", [(9, 5, 7, 8, 3), (4, 3, 5, 6, 8)])
def test_owner_rooted_chunk_broadcast_world2(tmp_path, m, n, s, p, nchunks):
    import oracle as O
    out = str(tmp_path / "c.npz")
    mp.spawn(_worker_chunks, args=(2, _free_port(), m, n, s, p, nchunks, out), nprocs=2, join=True)
    got = np.load(out)
    want = O.tprod_fast(O.gen_random_tensor(m, n, p, 21), O.gen_random_tensor(n, s, p, 22))
    assert np.array_equal(got["c1"].view(np.uint64), want[0].view(np.uint64))
    assert np.array_equal(got["c2"].view(np.uint64), want[1].view(np.uint64))


def test_column_chunk_plan():
    from paper_2212_14318_b200 import shard
    plan = shard.column_chunks(2048, 8, 8)
    assert [o for _, _, o in plan] == list(range(8)) and all(c1 - c0 == 256 for c0, c1, _ in plan)
    plan = shard.column_chunks(70, 8, 3)
    assert plan[0][0] == 0 and plan[-1][1] == 70 and all((c1 - c0) % 16 == 0 or c1 == 70 for c0, c1, _ in plan)
    assert [o for _, _, o in plan] == [j % 3 for j in range(len(plan))]
    assert shard.column_chunks(0, 8, 2) == []


def _cpu_freq_class():
    """FreqParallelTProduct with its three stages restated in numpy (the
    oracle's tube transforms; the paired per-frequency product of
    csrc/qt_ozaki.cu in complex arithmetic) and its exchange schedule as is."""
    import oracle as O
    from paper_2212_14318_b200 import distributed

    def cview(t):
        return t.numpy().view(np.complex128)

    class CpuFreq(distributed.FreqParallelTProduct):
        def k1(self, stream=None):
            if self.b1 > self.b0:
                y = O.qfft3_conj((cview(self.b[0]), cview(self.b[1])))
                cview(self.bh[0])[:], cview(self.bh[1])[:] = y
            if self.rows:
                y = O.qfft3_conj((cview(self.a[0]), cview(self.a[1])))
                cview(self.ah[0])[:], cview(self.ah[1])[:] = y

        def k2_prepare(self, stream=None):
            return True if self.ns else None

        def k2_multiply(self, h, stream=None):
            if h is None:
                return
            A1, A2, B1, B2 = cview(self.ac[0]), cview(self.ac[1]), cview(self.bc[0]), cview(self.bc[1])
            C1, C2 = cview(self.cc[0]), cview(self.cc[1])
            for t in range(self.s0, self.s1):
                k = self.freq[t]
                part = t if (self.p - k) % self.p == k else t ^ 1
                i, j = t - self.s0, part - self.s0
                C1[i] = A1[i] @ B1[i] - np.conj(A2[j]) @ B2[i]
                C2[i] = A2[i] @ B1[i] + np.conj(A1[j]) @ B2[i]

        def k3(self, stream=None):
            if self.rows:
                y = O.qifft3_conj((cview(self.c[0]), cview(self.c[1])))
                cview(self.c[0])[:], cview(self.c[1])[:] = y

    return CpuFreq


def _worker_freq(rank, world, port, m, n, s, p, out_path):
    """distributed.FreqParallelTProduct's exchange over gloo point-to-point
    ops (make_exchange), stages on the CPU: Â/B̂ row pieces to the slot
    owners, Ĉ pieces back to the row owners."""
    import sys
    sys.path.insert(0, ROOT)
    import oracle as O
    from paper_2212_14318_b200 import distributed, shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A = O.gen_random_tensor(m, n, p, 41)
    B = O.gen_random_tensor(n, s, p, 42)
    x = _cpu_freq_class()(m, n, s, p, rank, world, device="cpu")
    x.load_a(*A)
    x.load_b(*B)
    x.step(distributed.make_exchange(rank, dist))
    c = x.c.numpy().view(np.complex128)
    mb = -(-m // world)
    buf = np.zeros((2, p, mb, s), np.complex128)
    buf[:, :, :x.rows] = c
    tt = torch.from_numpy(buf.view(np.float64))
    gathered = [torch.zeros_like(tt) for _ in range(world)] if rank == 0 else None
    dist.gather(tt, gathered, dst=0)
    if rank == 0:
        out = np.zeros((2, p, m, s), np.complex128)
        for r, g in enumerate(gathered):
            r0, r1 = shard.row_slab(m, world, r)
            out[:, :, r0:r1] = g.numpy().view(np.complex128)[:, :, :r1 - r0]
        np.save(out_path, out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("m,n,s,p,world", [(9, 5, 6, 8, 2), (7, 3, 4, 7, 2), (5, 6, 3, 4, 3), (3, 2, 2, 2, 2)])
def test_freq_parallel_exchange(tmp_path, m, n, s, p, world):
    import oracle as O
    out = str(tmp_path / "c.npy")
    mp.spawn(_worker_freq, args=(world, _free_port(), m, n, s, p, out), nprocs=world, join=True)
    got = np.load(out)
    A = O.gen_random_tensor(m, n, p, 41)
    B = O.gen_random_tensor(n, s, p, 42)
    # the same stages on one rank: bitwise (every slot is computed identically)
    one = _cpu_freq_class()(m, n, s, p, 0, 1, device="cpu")
    one.load_a(*A)
    one.load_b(*B)
    one.step()
    assert np.array_equal(got.view(np.uint64), one.c.numpy().view(np.uint64))
    want = O.tprod_fast(A, B)
    assert O.rel_frob_error((got[0], got[1]), want) < 1e-13


def test_slot_ranges_keep_pairs_whole():
    from paper_2212_14318_b200 import shard
    for p in range(1, 70):
        assert sorted(shard.slot_freq(p, t) for t in range(p)) == list(range(p))
        for world in (1, 2, 3, 8):
            rs = shard.slot_ranges(p, world)
            assert rs[0][0] == 0 and rs[-1][1] == p and all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            pair_end = 2 * ((p - 1) // 2)
            assert all(not (b & 1 and b < pair_end) for r in rs for b in r)
            sizes = [t1 - t0 for t0, t1 in rs]
            assert max(sizes) - min(sizes) <= 2, (p, world, rs)


@pytest.mark.parametrize("m,n,s,p,world", [(9, 5, 6, 8, 2), (7, 3, 4, 7, 3), (5, 6, 3, 4, 3), (11, 4, 5, 6, 4),
                                           (3, 2, 2, 2, 2), (6, 4, 3, 5, 1)])
def test_freq_parallel_routing_tables(m, n, s, p, world):
    """The row tables of the fused exchange (FreqParallelTProduct.set_peers):
    every rank's frequency rows of Â/B̂, stored to the addresses its tables
    give (a memmove per row stands in for the routed K1 stores into the
    peers' stage buffers), and its rows of Ĉ, loaded from the addresses of
    its K3 table, reproduce the point-to-point exchange — so the stitched C
    equals the one-rank product bitwise."""
    import ctypes
    import oracle as O
    from paper_2212_14318_b200 import shard
    A = O.gen_random_tensor(m, n, p, 43)
    B = O.gen_random_tensor(n, s, p, 44)
    cls = _cpu_freq_class()
    ranks = [cls(m, n, s, p, r, world, device="cpu") for r in range(world)]
    bases = [x.stage_buffer.data_ptr() for x in ranks]
    for x in ranks:
        x.load_a(*A)
        x.load_b(*B)
        x.set_peers(bases)
        x.k1()  # into x.ah / x.bh, then "stored" row by row through the tables
        for key, src in (("a", x.ah), ("b", x.bh)):
            rowbytes = src[0, 0].numel() * 8
            if rowbytes == 0:
                continue
            for pl in (0, 1):
                for k in range(p):
                    ctypes.memmove(int(x.tables[key][pl][k]), src[pl, k].data_ptr(), rowbytes)
    for x in ranks:
        x.k2_multiply(x.k2_prepare())
    for x in ranks:
        rowbytes = x.c[0, 0].numel() * 8
        if rowbytes:
            for pl in (0, 1):
                for k in range(p):
                    ctypes.memmove(x.c[pl, k].data_ptr(), int(x.tables["c"][pl][k]), rowbytes)
        x.k3()
    one = cls(m, n, s, p, 0, 1, device="cpu")
    one.load_a(*A)
    one.load_b(*B)
    one.step()
    want = one.c.numpy().view(np.uint64)
    for x in ranks:
        r0, r1 = shard.row_slab(m, world, x.rank)
        assert np.array_equal(x.c.numpy().view(np.uint64), want[:, :, r0:r1]), x.rank
