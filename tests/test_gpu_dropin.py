"""GPU: the reference's own C++ test-suite, compiled UNMODIFIED against the
C++ drop-in (paper_2212_14318_b200/dropin/*.cpp replacing proj/src/tproduct.cpp
and proj/src/transform.cpp; the rest of the reference library unchanged),
run on the B200.  Built by __graft_entry__.build() where /root/reference
exists; the binaries travel in-tree.

* doctest suites (runner: tests/cpp/doctest.h): test_tproduct, test_transform,
  test_algebra, test_linalg, test_diag, test_io_bench — all must pass.
* acceptance.cpp (plain main, one PASS/FAIL line per criterion): every
  criterion except 2 must pass.  Criterion 2 asserts the CPU speed-up SHAPE of
  fast vs definitional at (20,20,20), p = 8..64 (acceptance.cpp:67-85); with
  both routes on the GPU the tiny calls are host-call-overhead bound, so the
  ratio is not the CPU's (the reference itself fails it on this pool's Xeon,
  SURVEY §4) — its line is reported, not asserted.
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


def _run(name, timeout=900):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        pytest.fail(f"{exe} not built (run __graft_entry__.build() where /root/reference exists)")
    return subprocess.run([exe], capture_output=True, text=True, timeout=timeout, cwd=os.path.dirname(exe))


@pytest.mark.parametrize("name", SUITES)
def test_reference_unit_tests_pass_on_dropin(name):
    r = _run(name)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stderr[-3000:]
    assert "| 0 failed" in r.stdout


def test_reference_acceptance_gate_on_dropin():
    r = _run("acceptance_dropin")
    print(r.stdout)
    lines = dict(re.findall(r"criterion (\d+): (PASS|FAIL)", r.stdout))
    assert len(lines) == 9, r.stdout + r.stderr
    for k, v in lines.items():
        if k != "2":
            assert v == "PASS", f"criterion {k}: {r.stdout}"
