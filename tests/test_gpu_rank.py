"""GPU: the per-rank multi-GPU drivers (csrc/qt_rank.cu) on one B200.

* `world` frequency-parallel ranks emulated in lockstep on one device
  (qt_rank_freq_emulate: the same partition and piece schedule as the NCCL
  exchange, every piece a device copy) stitch to tprod_fast bitwise — int8
  and fp64 stage 2, ragged partitions, p = 1 / odd / even;
* the real NCCL paths with a one-rank communicator (RankComm world 1): the
  row split (broadcast of B in place, then the slab product) and the
  frequency-parallel step, bitwise;
* non-finite input through the frequency-parallel step: its slots fall back
  to the fp64 kernels, as the single-GPU product does.
(Ranks whose kernels wait on each other are never run on one GPU; the
multi-process schedule itself is exercised over gloo on CPU.)
"""
import numpy as np
import pytest

import paper_2212_14318_b200 as qt
from paper_2212_14318_b200 import _native, distributed

pytestmark = pytest.mark.gpu


def bits_equal(x, y):
    return np.array_equal(np.ascontiguousarray(x).view(np.uint64), np.ascontiguousarray(y).view(np.uint64))


def dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x).view(np.float64)).cuda()


@pytest.mark.parametrize("m,n,s,p", [(150, 256, 520, 6), (97, 256, 512, 5), (130, 40, 70, 12), (33, 17, 40, 7),
                                     (20, 64, 300, 1), (5, 32, 9, 8)])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("fused", [False, True])
def test_freq_parallel_emulated_bitwise(m, n, s, p, world, fused):
    """fused: the exchange done by the transforms themselves — K1's routed
    stores into the other ranks' buffers, K3's routed loads from them (the
    row tables of qt_rank_freq_set_peers), lockstep order for the barriers."""
    import torch
    a = qt.gen_random_tensor(m, n, p, 91)
    b = qt.gen_random_tensor(n, s, p, 92)
    want = qt.tprod_fast(a, b)
    c1 = torch.full((p, m, 2 * s), float("nan"), dtype=torch.float64, device="cuda")
    c2 = torch.full_like(c1, float("nan"))
    distributed.emulate_freq(world, dev(a.t1), dev(a.t2), dev(b.t1), dev(b.t2), c1, c2, m, n, s, p, fused=fused)
    torch.cuda.synchronize()
    got1 = c1.cpu().numpy().view(np.complex128)
    got2 = c2.cpu().numpy().view(np.complex128)
    assert bits_equal(got1, want.t1) and bits_equal(got2, want.t2), (m, n, s, p, world)


@pytest.fixture(scope="module")
def comm1():
    c = distributed.RankComm(0, 1, 0)
    yield c
    c.close()


@pytest.mark.parametrize("m,n,s,p", [(150, 256, 520, 6), (130, 40, 70, 12), (64, 2048, 256, 4)])
def test_rows_world1_bitwise(comm1, m, n, s, p):
    import torch
    a = qt.gen_random_tensor(m, n, p, 11)
    b = qt.gen_random_tensor(n, s, p, 12)
    want = qt.tprod_fast(a, b)
    x = distributed.RowsTProduct(comm1, m, n, s, p)
    x.load_a(a.t1, a.t2)
    x.load_b(b.t1, b.t2)
    for _ in range(2):
        x.step()
        torch.cuda.synchronize()
        c1, c2 = x.result()
        assert bits_equal(c1, want.t1) and bits_equal(c2, want.t2)


@pytest.mark.parametrize("m,n,s,p", [(150, 256, 520, 6), (130, 40, 70, 12), (7, 32, 5, 3)])
def test_freq_world1_bitwise_and_nonfinite(comm1, m, n, s, p):
    import torch
    a = qt.gen_random_tensor(m, n, p, 13)
    b = qt.gen_random_tensor(n, s, p, 14)
    want = qt.tprod_fast(a, b)
    x = distributed.FreqTProduct(comm1, m, n, s, p)
    assert (x.a0, x.a1, x.b0, x.b1, x.slot0, x.slot1) == (0, m, 0, n, 0, p)
    x.load_a(a.t1, a.t2)
    x.load_b(b.t1, b.t2)
    for _ in range(2):
        x.step()
        torch.cuda.synchronize()
        c1, c2 = x.result()
        assert bits_equal(c1, want.t1) and bits_equal(c2, want.t2)
    b1 = b.t1.copy()
    b1[1, 2, 3] = float("inf")
    x.load_b(b1, b.t2)
    x.step()
    torch.cuda.synchronize()
    want = qt.tprod_fast(a, qt.CdTensor3(n, s, p, b1, b.t2))
    c1, c2 = x.result()
    assert np.array_equal(c1, want.t1, equal_nan=True) and np.array_equal(c2, want.t2, equal_nan=True)
    if _native.lib().qt_gemm_algo(m, n, s, p) == 1:
        assert x.nonfinite()
    x.close()


@pytest.mark.parametrize("ipc", [False, True])
def test_freq_fused_world1_bitwise(comm1, ipc):
    """The fused exchange through the real entry points at world 1 (own IPC
    handle; the device barrier is a no-op at one rank): bitwise, twice."""
    import torch
    m, n, s, p = 150, 256, 520, 6
    a = qt.gen_random_tensor(m, n, p, 15)
    b = qt.gen_random_tensor(n, s, p, 16)
    want = qt.tprod_fast(a, b)
    grp = distributed.IpcGroup(0, 1, 0) if ipc else comm1
    x = distributed.FreqTProduct(grp, m, n, s, p)
    x.load_a(a.t1, a.t2)
    x.load_b(b.t1, b.t2)
    x.set_peers([x.ipc_handle()])
    for _ in range(2):
        x.c.fill_(float("nan"))
        x.step()
        torch.cuda.synchronize()
        c1, c2 = x.result()
        assert bits_equal(c1, want.t1) and bits_equal(c2, want.t2)
    x.close()


def _ipc_worker(rank, world, port, m, n, s, p, out_path):
    """One of `world` processes sharing cuda:0: an IPC plan, the peers' buffers
    opened from their CUDA IPC handles, the three fused phases separated by
    host-side synchronisation (no kernel ever waits on another process)."""
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2212_14318_b200 as qt
    from paper_2212_14318_b200 import distributed
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    a = qt.gen_random_tensor(m, n, p, 17)
    b = qt.gen_random_tensor(n, s, p, 18)
    x = distributed.FreqTProduct(distributed.IpcGroup(rank, world, 0), m, n, s, p)
    x.load_a(a.t1, a.t2)
    x.load_b(b.t1, b.t2)
    handles = [None] * world
    dist.all_gather_object(handles, x.ipc_handle())
    x.set_peers(handles)
    for k in range(3):
        torch.cuda.synchronize()
        dist.barrier()
        x.phase(k)
    torch.cuda.synchronize()
    dist.barrier()
    c1, c2 = x.result()
    np.savez(f"{out_path}.{rank}.npz", c1=c1, c2=c2, a0=x.a0, a1=x.a1)
    dist.barrier()
    x.close()
    dist.destroy_process_group()


def test_freq_fused_two_processes_one_gpu(tmp_path):
    """Two processes on one GPU exchange their pieces through CUDA IPC
    mappings of each other's stage buffers (routed K1 stores / K3 loads): the
    stitched C equals tprod_fast bitwise.  The device barrier is replaced by
    host synchronisation here (kernels of two processes are never made to
    wait on each other on one GPU)."""
    import socket
    import torch.multiprocessing as mp
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    m, n, s, p = 150, 256, 520, 6
    out = str(tmp_path / "c")
    mp.spawn(_ipc_worker, args=(2, port, m, n, s, p, out), nprocs=2, join=True)
    a = qt.gen_random_tensor(m, n, p, 17)
    b = qt.gen_random_tensor(n, s, p, 18)
    want = qt.tprod_fast(a, b)
    for r in range(2):
        d = np.load(f"{out}.{r}.npz")
        a0, a1 = int(d["a0"]), int(d["a1"])
        assert bits_equal(d["c1"], want.t1[:, a0:a1]) and bits_equal(d["c2"], want.t2[:, a0:a1]), r
