"""QT3 tensor file I/O.

CPU: header validation (qt_qt3_probe, no GPU) against the reference's
parse_tensor error kinds (test_io_bench.cpp:79-135).  GPU: bit-exact
file <-> device-plane round trips against the reference's own writer
(tests/golden/ref_gen_3x2x4_seed9.qt3) and serialiser."""
import os

import numpy as np
import pytest

import oracle as O
import paper_2212_14318_b200 as qt
from paper_2212_14318_b200 import tensor_io

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN_QT3 = os.path.join(HERE, "golden", "ref_gen_3x2x4_seed9.qt3")


def test_golden_file_is_the_reference_serialisation():
    t = O.gen_random_tensor(3, 2, 4, 9)
    assert open(GOLDEN_QT3, "rb").read() == O.qt3_bytes(*t)
    assert tensor_io.probe(GOLDEN_QT3) == (3, 2, 4)


def _bad(tmp_path, name, data):
    p = tmp_path / name
    p.write_bytes(bytes(data))
    return str(p)


def test_probe_rejects_malformed_headers_with_reference_kinds(tmp_path):
    good = bytearray(O.qt3_bytes(*O.gen_random_tensor(2, 2, 2, 5)))
    cases = []
    b = bytearray(good); b[1] = ord("X"); cases.append(("BadMagic", b))
    b = bytearray(good[:-1]); cases.append(("Truncated", b))
    b = bytearray(good); b[4] = 3; cases.append(("Truncated", b))             # dims vs length
    b = bytearray(good); b[4:12] = b"\xff" * 8; cases.append(("DimOverflow", b))
    b = bytearray(good); b[12:20] = b"\x00" * 8; cases.append(("DimOverflow", b))
    cases.append(("Truncated", bytearray(good[:10])))                          # short header, good magic
    cases.append(("BadMagic", bytearray(b"QT")))
    for k, (kind, data) in enumerate(cases):
        path = _bad(tmp_path, f"bad{k}.qt3", data)
        with pytest.raises(tensor_io.TensorIoError) as ei:
            tensor_io.probe(path)
        assert ei.value.kind == kind, (k, kind, str(ei.value))
        if O.ref_available():  # the reference agrees on the kind
            assert O.ref_read_tensor(path) == {"BadMagic": 6, "Truncated": 7, "DimOverflow": 8}[kind]
    with pytest.raises(tensor_io.TensorIoError) as ei:
        tensor_io.probe(str(tmp_path / "missing.qt3"))
    assert ei.value.kind == "Io"


@pytest.mark.gpu
def test_gpu_reads_reference_file_bitwise():
    t = tensor_io.read_tensor(GOLDEN_QT3)
    w1, w2 = O.gen_random_tensor(3, 2, 4, 9)
    assert np.array_equal(t.t1.view(np.uint64), w1.view(np.uint64))
    assert np.array_equal(t.t2.view(np.uint64), w2.view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,p", [(3, 2, 4), (1, 1, 1), (64, 64, 600)])  # the last spans two 64 MB chunks
def test_gpu_write_read_round_trip_bitwise(tmp_path, m, n, p):
    t = qt.gen_random_tensor(m, n, p, 77)
    path = str(tmp_path / "t.qt3")
    tensor_io.write_tensor(path, t)
    assert open(path, "rb").read() == O.qt3_bytes(t.t1, t.t2)
    back = tensor_io.read_tensor(path)
    assert np.array_equal(back.t1.view(np.uint64), t.t1.view(np.uint64))
    assert np.array_equal(back.t2.view(np.uint64), t.t2.view(np.uint64))


@pytest.mark.gpu
def test_gpu_read_feeds_the_tproduct(tmp_path):
    """A file streamed into HBM is directly the T-product's input layout."""
    a = qt.gen_random_tensor(20, 12, 8, 1)
    b = qt.gen_random_tensor(12, 9, 8, 2)
    pa, pb = str(tmp_path / "a.qt3"), str(tmp_path / "b.qt3")
    tensor_io.write_tensor(pa, a)
    tensor_io.write_tensor(pb, b)
    import torch
    a1, a2, m, n, p = tensor_io.read_tensor_device(pa)
    b1, b2, _, s, _ = tensor_io.read_tensor_device(pb)
    c1 = torch.empty((p, m, 2 * s), dtype=torch.float64, device="cuda")
    c2 = torch.empty_like(c1)
    qt.tprod_fast_device(a1, a2, b1, b2, c1, c2, m, n, s, p)
    torch.cuda.synchronize()
    want = qt.tprod_fast(a, b)
    assert np.array_equal(c1.cpu().numpy().view(np.complex128), want.t1)
