"""CPU: the C-ABI library loads and exports every symbol include/*.h declares;
host-only entry points (seeded generators) agree with the oracle.  No compute
entry point is called here (no GPU in this container)."""
import ctypes
import os
import re

import numpy as np

import oracle as O
from paper_2212_14318_b200 import _native
from paper_2212_14318_b200.configs import CONFIGS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    inc = os.path.join(ROOT, "include")
    for fn in os.listdir(inc):
        if fn.endswith(".h"):
            src = open(os.path.join(inc, fn)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            syms.update(re.findall(r"\b(qt_[a-z0-9_]+)\s*\(", src))
    return syms


def test_library_exports_every_declared_symbol():
    L = _native.lib()
    syms = declared_symbols()
    assert len(syms) >= 13
    for s in syms:
        assert hasattr(L, s), s
        assert s in _native.SIGNATURES, f"{s} has no ctypes signature"
    assert L.qt_abi_version() == 2
    assert L.qt_last_error() == b""


def test_no_symbol_outside_the_header_is_bound():
    assert set(_native.SIGNATURES) == declared_symbols()


def test_library_is_sm100a_only():
    data = open(_native.LIB_PATH, "rb").read()
    assert b"sm_100a" in data


def test_derive_seed_matches_oracle():
    for base, stream in [(42, 0), (42, 1), (42, 9), (7, 123)]:
        assert _native.lib().qt_derive_seed(base, stream) == O.derive_seed(base, stream)


def test_generator_bitwise_equals_reference_generator():
    from paper_2212_14318_b200 import gen_random_tensor
    for (m, n, p, seed) in [(4, 5, 3, 7), (1, 1, 1, 1), (32, 32, 16, 99)]:
        t = gen_random_tensor(m, n, p, seed)
        w1, w2 = O.gen_random_tensor(m, n, p, seed)
        assert np.array_equal(t.t1.view(np.uint64), w1.view(np.uint64))
        assert np.array_equal(t.t2.view(np.uint64), w2.view(np.uint64))


def test_generator_distributions_equal_oracle_restatement():
    """All three BASELINE input distributions (uniform, normal, pure-quaternion
    RGB): the library's generator equals the oracle's restatement bitwise (the
    reference arm of bench.py builds its inputs from the latter)."""
    from paper_2212_14318_b200 import gen_tensor
    for dist, scale in ((0, 1.0), (1, 1.0), (1, 1.0 / np.sqrt(1920.0)), (2, 1.0)):
        for (m, n, p, seed) in [(4, 5, 3, 7), (1, 1, 1, 1), (17, 9, 6, 12345)]:
            t = gen_tensor(m, n, p, seed, dist, scale)
            w1, w2 = O.gen_tensor(dist, m, n, p, seed, scale)
            assert np.array_equal(t.t1.view(np.uint64), w1.view(np.uint64)), (dist, m, n, p)
            assert np.array_equal(t.t2.view(np.uint64), w2.view(np.uint64)), (dist, m, n, p)


def test_config_table_is_standalone():
    """bench.py's reference arm loads configs.py by path, without the product
    package or its library: the module must not import either."""
    import importlib.util
    import subprocess
    import sys
    code = ("import importlib.util, sys\n"
            "spec = importlib.util.spec_from_file_location('cfgs', %r)\n"
            "m = importlib.util.module_from_spec(spec); sys.modules['cfgs'] = m; spec.loader.exec_module(m)\n"
            "assert not any(k.startswith('paper_2212_14318_b200') for k in sys.modules)\n"
            "print([m.CONFIGS[c].seeds() for c in (1, 5)])\n") % os.path.join(ROOT, "paper_2212_14318_b200",
                                                                                 "configs.py")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    want = [CONFIGS[c].seeds() for c in (1, 5)]
    assert r.stdout.strip() == str(want)


def test_generator_rejects_zero_dims():
    buf = np.zeros(8)
    rc = _native.lib().qt_gen_tensor_f64(0, 0, 1, 1, 1, 1.0, buf.ctypes.data, buf.ctypes.data)
    assert rc == _native.QT_EINVAL


def test_config_inputs_match_fixture_checksums(cfg_golden):
    """The generators behind the five BASELINE configs are the ones the golden
    reference outputs were computed from (small configs only here: 1, 3)."""
    from paper_2212_14318_b200 import make_inputs
    for c in (1, 3):
        a, b = make_inputs(CONFIGS[c])
        chk = np.array([np.sum(a.t1.real), np.sum(a.t1.imag), np.sum(a.t2.real), np.sum(a.t2.imag)])
        assert np.array_equal(chk, cfg_golden[f"cfg{c}_chkA"])
        assert list(CONFIGS[c].seeds()) == [int(v) for v in cfg_golden[f"cfg{c}_seeds"]]


def test_dropin_binaries_link_against_the_product_library():
    """The reference's unit tests built against the C++ drop-in resolve
    libqtensor_b200.so in-tree (no GPU needed to check the link)."""
    import subprocess
    import pytest
    bindir = os.path.join(ROOT, "paper_2212_14318_b200", "dropin", "bin")
    if not os.path.isdir(bindir):
        pytest.skip("drop-in binaries not built here")
    for name in os.listdir(bindir):
        out = subprocess.run(["ldd", os.path.join(bindir, name)], capture_output=True, text=True).stdout
        assert "libqtensor_b200.so" in out and "not found" not in out, out
