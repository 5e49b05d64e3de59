"""Full-tensor parity of the B200 T-product against the reference itself
(SURVEY §8(d) parity protocol).

The reference's own tprod_fast (oracle/_ref: /root/reference's sources
compiled unmodified by oracle/Makefile, namespace-renamed) runs here on every
host core, one (row x column) tile of C per thread.  A tile is bitwise the
matching block of the reference's full result (rows of C depend only on rows
of A, columns only on columns of B; SURVEY probe B9), so the stitched tiles ARE
the reference's C.  Bars: relative Frobenius error <= 1e-12 (BASELINE.json).

* configs 2, 3 and 4: the whole C;
* config 5: 32 full-width rows — the first / last rows of every 1/2/4/8-GPU
  row shard (boundaries at multiples of 256) plus seeded random rows;
* a negative control: with sigma(k) = k forced into stage 2
  ($QTB_DEBUG_NO_REFLECT=1, fp64 path) the same comparison must FAIL.
"""
import os
import subprocess
import sys
import threading

import numpy as np
import pytest

import oracle as O
import paper_2212_14318_b200 as qt

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (make -C oracle ref)")


def ref_tiles(a, b, rows, cols, row_idx=None):
    """The reference tprod_fast of A[row_idx] * B, as rows x cols tiles run in
    parallel (one host thread each; ctypes releases the GIL)."""
    a1, a2 = a
    if row_idx is not None:
        a1, a2 = a1[:, row_idx], a2[:, row_idx]
    p, m, _ = a1.shape
    s = b[0].shape[2]
    rs = np.array_split(np.arange(m), rows)
    cs = np.array_split(np.arange(s), cols)
    c1 = np.empty((p, m, s), np.complex128)
    c2 = np.empty_like(c1)
    errors = []

    def run(ri, ci):
        try:
            r0, r1 = ri[0], ri[-1] + 1
            q0, q1 = ci[0], ci[-1] + 1
            at = (np.ascontiguousarray(a1[:, r0:r1]), np.ascontiguousarray(a2[:, r0:r1]))
            bt = (np.ascontiguousarray(b[0][:, :, q0:q1]), np.ascontiguousarray(b[1][:, :, q0:q1]))
            t1, t2 = O.ref_tprod_fast(at, bt)
            c1[:, r0:r1, q0:q1] = t1
            c2[:, r0:r1, q0:q1] = t2
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    th = [threading.Thread(target=run, args=(ri, ci)) for ri in rs if len(ri) for ci in cs if len(ci)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    return c1, c2


def grid_for(m, s):
    """(row tiles, column tiles) ~ the host's cores, rows first (every column
    tile repeats the transforms of its rows of A)."""
    n = max(1, os.cpu_count() or 1)
    rows = min(m, n)
    cols = max(1, min(s, n // rows))
    return rows, cols


@needs_ref
@pytest.mark.parametrize("c", [1, 2, 3, 4])
def test_full_tensor_matches_reference(c):
    cfg = qt.CONFIGS[c]
    a, b = qt.make_inputs(cfg)
    got = qt.tprod_fast(a, b)
    want = ref_tiles((a.t1, a.t2), (b.t1, b.t2), *grid_for(cfg.m, cfg.s))
    err = O.rel_frob_error((got.t1, got.t2), want)
    print(f"config {c}: full C ({cfg.m} x {cfg.s} x {cfg.p}) vs reference tprod_fast: {err:.3e}")
    assert err <= 1e-12, err


def config5_rows():
    """32 rows of config 5: both sides of every 1/2/4/8-GPU shard boundary
    (multiples of 256), the first and last rows, and seeded random rows."""
    rows = {0, 1, 2046, 2047}
    for b in range(256, 2048, 256):
        rows |= {b - 1, b}
    rng = np.random.default_rng(55)
    while len(rows) < 32:
        rows.add(int(rng.integers(0, 2048)))
    return np.array(sorted(rows))


@needs_ref
def test_config5_rows_match_reference():
    cfg = qt.CONFIGS[5]
    a, b = qt.make_inputs(cfg)
    got = qt.tprod_fast(a, b)  # the whole product through the host C-ABI (int8 stage 2)
    rows = config5_rows()
    assert len(rows) >= 32
    ncpu = max(1, os.cpu_count() or 1)
    want = ref_tiles((a.t1, a.t2), (b.t1, b.t2), 1, min(ncpu, 16), row_idx=rows)
    err = O.rel_frob_error((got.t1[:, rows], got.t2[:, rows]), want)
    print(f"config 5: {len(rows)} full rows vs reference tprod_fast: {err:.3e}")
    assert err <= 1e-12, err


@needs_ref
def test_negative_control_sigma_identity_fails():
    """sigma(k) = k in stage 2 (forced through a debug switch, fp64 DMMA path):
    the same parity check must fail by many orders of magnitude, and pass
    again without the switch (the switch is read once per process, so both
    run in subprocesses)."""
    code = ("import sys; sys.path.insert(0, %r)\n"
            "import oracle as O, paper_2212_14318_b200 as qt\n"
            "a = qt.gen_random_tensor(40, 24, 12, 3); b = qt.gen_random_tensor(24, 30, 12, 4)\n"
            "c = qt.tprod_fast(a, b)\n"
            "print(O.rel_frob_error((c.t1, c.t2), O.ref_tprod_fast((a.t1, a.t2), (b.t1, b.t2))))\n") % ROOT
    errs = {}
    for flag in ("1", "0"):
        env = {**os.environ, "QTB_DEBUG_NO_REFLECT": flag, "QTB_OZAKI": "0"}
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env)
        assert r.returncode == 0, r.stderr[-2000:]
        errs[flag] = float(r.stdout.strip().splitlines()[-1])
    assert errs["0"] <= 1e-12, errs
    assert errs["1"] > 1e-3, errs
