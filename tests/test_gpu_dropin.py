"""GPU: the reference's own C++ test-suite, compiled UNMODIFIED against the
C++ drop-in (paper_2212_14318_b200/dropin/*.cpp replacing proj/src/tproduct.cpp
and proj/src/transform.cpp; the rest of the reference library unchanged),
run on the B200.  Built by __graft_entry__.build() where /root/reference
exists; the binaries travel in-tree.

* doctest suites (runner: tests/cpp/doctest.h): test_tproduct, test_transform,
  test_algebra, test_linalg, test_diag, test_io_bench — all must pass.
* acceptance.cpp (plain main, one PASS/FAIL line per criterion): all nine
  criteria must pass.  The drop-in's tprod_naive is the reference's own CPU
  definition by default (an independent oracle for the GPU product), so
  criterion 2 — the speed-up of fast over definitional growing with p and
  >= 8x at p = 64 (acceptance.cpp:67-85) — measures GPU tprod_fast against it.
* test_tproduct again with the definitional product on the GPU as well
  (QTB_DROPIN_NAIVE=gpu).
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2212_14318_b200", "dropin", "bin")

pytestmark = pytest.mark.gpu

SUITES = ["test_tproduct_dropin", "test_transform_dropin", "test_tproduct_fulldropin", "test_algebra_dropin",
          "test_linalg_dropin", "test_diag_dropin", "test_io_bench_dropin"]


def _run(name, timeout=900, env=None):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        pytest.fail(f"{exe} not built (run __graft_entry__.build() where /root/reference exists)")
    return subprocess.run([exe], capture_output=True, text=True, timeout=timeout, cwd=os.path.dirname(exe),
                          env={**os.environ, **(env or {})})


@pytest.mark.parametrize("name", SUITES)
def test_reference_unit_tests_pass_on_dropin(name):
    r = _run(name)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stderr[-3000:]
    assert "| 0 failed" in r.stdout


def test_reference_tproduct_suite_with_gpu_definitional_product():
    r = _run("test_tproduct_dropin", env={"QTB_DROPIN_NAIVE": "gpu"})
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0 and "| 0 failed" in r.stdout, r.stderr[-3000:]


def test_reference_acceptance_gate_on_dropin():
    r = _run("acceptance_dropin")
    print(r.stdout)
    lines = dict(re.findall(r"criterion (\d+): (PASS|FAIL)", r.stdout))
    assert len(lines) == 9, r.stdout + r.stderr
    for k, v in lines.items():
        assert v == "PASS", f"criterion {k}: {r.stdout}"
