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


def _freq_rank_cpu(m, n, s, p, world, rank, A, B, exchange):
    """One frequency-parallel rank with the LIBRARY's partition and exchange
    schedule (qt_rank_partition / qt_rank_freq_schedule, csrc/qt_rank.cu) and
    its buffers laid out as the C++ driver's, the stages restated on the CPU
    (the oracle's tube transforms; the paired per-frequency product of SURVEY
    §8(a) in complex arithmetic).  `exchange(sends, recvs)` moves the pieces
    (lists of (peer, array view) in transfer order)."""
    import oracle as O
    from paper_2212_14318_b200 import distributed, shard
    a0, a1, b0, b1, t0, t1 = distributed.partition(m, n, p, world, rank)
    ra, rb, ns = a1 - a0, b1 - b0, t1 - t0
    ah = np.zeros((2, p, ra, n), np.complex128)
    bh = np.zeros((2, p, rb, s), np.complex128)
    ac = np.zeros((2, ns, m, n), np.complex128)
    bc = np.zeros((2, ns, n, s), np.complex128)
    cc = np.zeros((2, ns, m, s), np.complex128)
    c = np.zeros((2, p, ra, s), np.complex128)
    if rb:
        bh[0], bh[1] = O.qfft3_conj((np.ascontiguousarray(B[0][:, b0:b1]), np.ascontiguousarray(B[1][:, b0:b1])))
    if ra:
        ah[0], ah[1] = O.qfft3_conj((np.ascontiguousarray(A[0][:, a0:a1]), np.ascontiguousarray(A[1][:, a0:a1])))

    def views(part, send):
        out = []
        for peer, slot, pl, r0, rows in distributed.schedule(m, n, s, p, world, rank, part, send):
            k = shard.slot_freq(p, slot)
            if (part == "c") != send:  # this side holds rows of every frequency
                buf = {"a": ah, "b": bh, "c": c}[part]
                v = buf[pl, k]
                assert v.shape[0] == rows
            else:  # this side owns the slot
                buf = {"a": ac, "b": bc, "c": cc}[part]
                v = buf[pl, slot - t0, r0:r0 + rows]
            out.append((peer, v))
        return out

    exchange(views("b", True), views("b", False))
    exchange(views("a", True), views("a", False))
    for t in range(t0, t1):
        k = shard.slot_freq(p, t)
        sk = (p - k) % p
        part = t if sk == k else t ^ 1
        i, j = t - t0, part - t0
        cc[0, i] = ac[0, i] @ bc[0, i] - np.conj(ac[1, j]) @ bc[1, i]
        cc[1, i] = ac[1, i] @ bc[0, i] + np.conj(ac[0, j]) @ bc[1, i]
    exchange(views("c", True), views("c", False))
    if ra:
        c[0], c[1] = O.qifft3_conj((c[0], c[1]))
    return a0, a1, c


def _local_exchange(rank):
    def ex(sends, recvs):
        src = [v for peer, v in sends if peer == rank]
        dst = [v for peer, v in recvs if peer == rank]
        assert len(src) == len(dst) == len(sends) == len(recvs)
        for a, b in zip(src, dst):
            b[...] = a
    return ex


def _worker_freq(rank, world, port, m, n, s, p, out_path):
    """The frequency-parallel schedule of csrc/qt_rank.cu over gloo
    point-to-point ops (the C++ driver's NCCL send/recv groups), stages on the
    CPU: Â/B̂ row pieces to the slot owners, Ĉ pieces back to the row owners."""
    import sys
    sys.path.insert(0, ROOT)
    import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A = O.gen_random_tensor(m, n, p, 41)
    B = O.gen_random_tensor(n, s, p, 42)

    def exchange(sends, recvs):
        for peer, v in sends:
            assert v.flags["C_CONTIGUOUS"]
        local = _local_exchange(rank)
        ls = [(q, v) for q, v in sends if q == rank]
        lr = [(q, v) for q, v in recvs if q == rank]
        local(ls, lr)
        ops, keep = [], []
        for q, v in sends:
            if q != rank:
                t = torch.from_numpy(v.view(np.float64).reshape(-1))
                keep.append(t)
                ops.append(dist.P2POp(dist.isend, t, q))
        rbufs = []
        for q, v in recvs:
            if q != rank:
                t = torch.empty(v.size * 2, dtype=torch.float64)
                rbufs.append((t, v))
                ops.append(dist.P2POp(dist.irecv, t, q))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        for t, v in rbufs:
            v[...] = t.numpy().view(np.complex128).reshape(v.shape)

    a0, a1, c = _freq_rank_cpu(m, n, s, p, world, rank, A, B, exchange)
    mb = -(-m // world)
    buf = np.zeros((2, p, mb, s), np.complex128)
    buf[:, :, :a1 - a0] = c
    tt = torch.from_numpy(buf.view(np.float64))
    gathered = [torch.zeros_like(tt) for _ in range(world)] if rank == 0 else None
    dist.gather(tt, gathered, dst=0)
    if rank == 0:
        from paper_2212_14318_b200 import shard
        out = np.zeros((2, p, m, s), np.complex128)
        for r, g in enumerate(gathered):
            r0, r1 = shard.row_slab(m, world, r)
            out[:, :, r0:r1] = g.numpy().view(np.complex128)[:, :, :r1 - r0]
        np.save(out_path, out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("m,n,s,p,world", [(9, 5, 6, 8, 2), (7, 3, 4, 7, 2), (5, 6, 3, 4, 3), (3, 2, 2, 2, 2),
                                           (11, 4, 5, 6, 4)])
def test_freq_parallel_exchange(tmp_path, m, n, s, p, world):
    """The library's frequency-parallel partition + schedule, executed over
    gloo by `world` processes, stitches to the one-rank result bitwise (every
    slot is computed identically) and to the reference within 1e-13."""
    import oracle as O
    out = str(tmp_path / "c.npy")
    mp.spawn(_worker_freq, args=(world, _free_port(), m, n, s, p, out), nprocs=world, join=True)
    got = np.load(out)
    A = O.gen_random_tensor(m, n, p, 41)
    B = O.gen_random_tensor(n, s, p, 42)
    _, _, one = _freq_rank_cpu(m, n, s, p, 1, 0, A, B, _local_exchange(0))
    assert np.array_equal(got.view(np.uint64), one.view(np.uint64))
    want = O.tprod_fast(A, B)
    assert O.rel_frob_error((got[0], got[1]), want) < 1e-13


def test_library_partition_equals_shard_rules():
    """qt_rank_partition (C++) and shard.row_slab / shard.slot_ranges agree."""
    from paper_2212_14318_b200 import distributed, shard
    for m, n, p in [(2048, 2048, 32), (1080, 1920, 64), (16, 16, 4096), (9, 5, 8), (3, 7, 1), (5, 2, 2), (1, 1, 9)]:
        for world in (1, 2, 3, 4, 5, 8):
            for r in range(world):
                a0, a1, b0, b1, t0, t1 = distributed.partition(m, n, p, world, r)
                assert (a0, a1) == shard.row_slab(m, world, r)
                assert (b0, b1) == shard.row_slab(n, world, r)
                assert (t0, t1) == shard.slot_ranges(p, world)[r], (m, n, p, world, r)


def test_library_schedule_pairs_every_piece():
    """Every send of the library's schedule has exactly one matching receive
    (same peer pair, position and size), for every part and world."""
    from paper_2212_14318_b200 import distributed
    for m, n, s, p in [(9, 5, 6, 8), (2, 3, 4, 7), (5, 6, 3, 1), (13, 4, 5, 6)]:
        for world in (1, 2, 3, 4):
            for part in "abc":
                snd = [distributed.schedule(m, n, s, p, world, r, part, True) for r in range(world)]
                rcv = [distributed.schedule(m, n, s, p, world, r, part, False) for r in range(world)]
                for src in range(world):
                    for dst in range(world):
                        a = [x for x in snd[src] if x[0] == dst]
                        b = [x for x in rcv[dst] if x[0] == src]
                        assert len(a) == len(b), (m, n, s, p, world, part, src, dst)
                        for x, y in zip(a, b):
                            assert x[1:3] == y[1:3] and x[4] == y[4]


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
