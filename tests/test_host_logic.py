"""CPU: host-side logic of the Python mirror (argument checks that fire before
any device work, the pairing table, flop model, config metadata)."""
import numpy as np
import pytest

import oracle as O
import paper_2212_14318_b200 as qt
from paper_2212_14318_b200 import shard


def test_slice_reflect_pinned():  # test_tproduct.cpp:47-58
    table = {(0, 1): 0, (0, 2): 0, (1, 2): 1, (0, 3): 0, (1, 3): 2, (2, 3): 1,
             (0, 4): 0, (1, 4): 3, (2, 4): 2, (3, 4): 1}
    for (i, p), want in table.items():
        assert qt.slice_reflect(i, p) == want


def test_flops_estimate_matches_reference():
    for m, n, s, p in [(1, 1, 1, 1), (1, 1, 1, 2), (3, 4, 5, 7), (20, 20, 20, 64), (2048, 2048, 2048, 32)]:
        f = qt.flops_estimate(m, n, s, p)
        assert [f.fast_mults, f.fast_transform_flops, f.naive_mults, f.naive_adds] == O.flops_estimate(m, n, s, p)
    with pytest.raises(ValueError):
        qt.flops_estimate(0, 1, 1, 1)


def test_dimension_mismatch_raises_before_device_work():  # tproduct.cpp:76-77
    a = qt.CdTensor3(2, 2, 2)
    with pytest.raises(ValueError):
        qt.tprod_fast(a, qt.CdTensor3(3, 2, 2))
    with pytest.raises(ValueError):
        qt.tprod_fast(a, qt.CdTensor3(2, 2, 3))


def test_cdtensor_layout_is_reference_layout():  # transform.hpp:35-37
    t = qt.CdTensor3(3, 4, 5)
    flat = t.t1.reshape(-1)
    t.set_qat(2, 1, 3, (1.0, 2.0, 3.0, 4.0))
    assert flat[t.idx(2, 1, 3)] == 1 + 2j
    assert t.qat(2, 1, 3) == (1.0, 2.0, 3.0, 4.0)
    assert t.t2.reshape(-1)[(3 * 3 + 2) * 4 + 1] == 3 + 4j


def test_config_work_model():
    c5 = qt.CONFIGS[5]
    assert c5.flops_gemm == 32.0 * 2048 ** 3 * 32
    assert c5.bytes_gemm == 3 * 32 * 2048 * 2048 * 32
    assert qt.CONFIGS[4].m == 1080 and qt.CONFIGS[4].n == 1920 and qt.CONFIGS[4].s == 64


@pytest.mark.parametrize("m,world", [(2048, 8), (1080, 8), (7, 4), (3, 8), (256, 1), (1, 2)])
def test_row_slabs_partition_rows(m, world):
    got = [shard.row_slab(m, world, r) for r in range(world)]
    rows = [i for lo, hi in got for i in range(lo, hi)]
    assert rows == list(range(m))
    sizes = [hi - lo for lo, hi in got]
    assert max(sizes) - min(s for s in sizes if s) <= max(1, -(-m // world))
