"""GPU: the reference's own C++ unit tests, compiled UNMODIFIED against the C++
drop-in (paper_2212_14318_b200/dropin/*.cpp replacing proj/src/tproduct.cpp
and proj/src/transform.cpp), run on the B200.  The binaries are built by
__graft_entry__.build() where /root/reference exists and travel in-tree."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2212_14318_b200", "dropin", "bin")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["test_tproduct_dropin", "test_transform_dropin", "test_tproduct_fulldropin"])
def test_reference_unit_tests_pass_on_dropin(name):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        pytest.fail(f"{exe} not built (run __graft_entry__.build() where /root/reference exists)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "0 failed" in r.stdout
