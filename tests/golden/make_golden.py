"""Generate tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref, compiled
from /root/reference's own sources by `make -C oracle ref`).

Run here (the container that has /root/reference):  python tests/golden/make_golden.py
The GPU box has no /root/reference; it only reads the committed .npz files.

Fixture contents
* small.npz    — full inputs and reference outputs (tprod_fast, tprod_naive,
                 qfft3_conj, qifft3_conj) for small seeded cases covering p = 1,
                 even/odd/prime p and degenerate m, n, s = 1.
* ref_gen_3x2x4_seed9.qt3 — gen_random_tensor(3, 2, 4, 9) written by the
                 reference's write_tensor (QT3 format, tensor_io.hpp:16-20).
* configs.npz  — per BASELINE config: the input seeds, an input checksum, and
                 reference tprod_fast outputs on sampled (row-set x column-set)
                 tiles.  Row i / column j of C depend only on row i of A /
                 column j of B, and the reference's tile runs are bitwise
                 identical to its full run (verified below for config 1), so a
                 tile is an exact sample of the full reference output.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_2212_14318_b200.configs import CONFIGS  # noqa: E402
from paper_2212_14318_b200.tproduct import gen_tensor  # noqa: E402  (host RNG, no GPU)

HERE = os.path.dirname(os.path.abspath(__file__))

SMALL = [  # (m, n, s, p, seedA, seedB)
    (5, 4, 3, 6, 101, 102), (2, 3, 2, 1, 103, 104), (3, 2, 4, 7, 105, 106), (4, 3, 5, 8, 107, 108),
    (1, 1, 1, 5, 109, 110), (8, 8, 8, 12, 111, 112), (6, 5, 7, 11, 113, 114), (1, 7, 1, 4, 115, 116),
    (7, 1, 6, 9, 117, 118), (3, 3, 3, 2, 119, 120), (9, 6, 3, 16, 121, 122), (4, 5, 6, 97, 123, 124),
    (3, 4, 2, 100, 125, 126), (17, 19, 23, 10, 127, 128),
]


def checksum(t) -> np.ndarray:
    return np.array([np.sum(t.t1.real), np.sum(t.t1.imag), np.sum(t.t2.real), np.sum(t.t2.imag)])


def tiles_for(cfg, rng):
    """Row sets cover the first/last rows and every 1/2/4/8-way shard boundary."""
    m, s = cfg.m, cfg.s
    rows = {0, m - 1}
    for g in (2, 4, 8):
        slab = -(-m // g)
        for k in range(1, g):
            b = k * slab
            if b < m:
                rows.update({b - 1, b})
    rows = sorted(rows)
    extra = sorted(set(rng.choice(m, size=min(m, 4), replace=False).tolist()) - set(rows))
    cols = sorted(set([0, s - 1] + rng.choice(s, size=min(s, 4), replace=False).tolist()))
    return np.array(rows + extra, np.int64), np.array(cols, np.int64)


def main():
    assert O.ref_available(), "build oracle/_ref first: make -C oracle ref"
    out = {}
    for idx, (m, n, s, p, sa, sb) in enumerate(SMALL):
        a = O.ref_gen_random_tensor(m, n, p, sa)
        b = O.ref_gen_random_tensor(n, s, p, sb)
        out[f"c{idx}_shape"] = np.array([m, n, s, p])
        out[f"c{idx}_a1"], out[f"c{idx}_a2"] = a
        out[f"c{idx}_b1"], out[f"c{idx}_b2"] = b
        out[f"c{idx}_fast1"], out[f"c{idx}_fast2"] = O.ref_tprod_fast(a, b)
        out[f"c{idx}_naive1"], out[f"c{idx}_naive2"] = O.ref_tprod_naive(a, b)
        out[f"c{idx}_fa1"], out[f"c{idx}_fa2"] = O.ref_qfft3_conj(a)
        out[f"c{idx}_ia1"], out[f"c{idx}_ia2"] = O.ref_qifft3_conj(a)
    out["ncases"] = np.array(len(SMALL))
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)

    rng = np.random.default_rng(20241019)
    cfg_out = {}
    for c, cfg in CONFIGS.items():
        sa, sb = cfg.seeds()
        a = gen_tensor(cfg.m, cfg.n, cfg.p, sa, cfg.dist_a, cfg.scale_a)
        b = gen_tensor(cfg.n, cfg.s, cfg.p, sb, cfg.dist_b, cfg.scale_b)
        rows, cols = tiles_for(cfg, rng)
        a_t = (a.t1[:, rows, :], a.t2[:, rows, :])
        b_t = (b.t1[:, :, cols], b.t2[:, :, cols])
        c1, c2 = O.ref_tprod_fast(a_t, b_t)
        cfg_out[f"cfg{c}_seeds"] = np.array([sa, sb], np.uint64)
        cfg_out[f"cfg{c}_chkA"] = checksum(a)
        cfg_out[f"cfg{c}_chkB"] = checksum(b)
        cfg_out[f"cfg{c}_rows"] = rows
        cfg_out[f"cfg{c}_cols"] = cols
        # store every slice for p <= 64; for long tubes a slice sample plus the
        # per-entry sum and sum of squares over all slices (catches any slice)
        sl = np.arange(cfg.p) if cfg.p <= 64 else np.unique(np.concatenate(
            [[0, 1, cfg.p // 2, cfg.p - 1], rng.choice(cfg.p, size=28, replace=False)]))
        cfg_out[f"cfg{c}_slices"] = sl
        cfg_out[f"cfg{c}_c1"] = c1[sl]
        cfg_out[f"cfg{c}_c2"] = c2[sl]
        cfg_out[f"cfg{c}_sum"] = np.stack([c1.sum(0), c2.sum(0)])
        cfg_out[f"cfg{c}_sumsq"] = np.stack([(np.abs(c1) ** 2).sum(0), (np.abs(c2) ** 2).sum(0)])
        if c == 1:  # tile == full-run sample, bitwise (the property the sampling relies on)
            f1, f2 = O.ref_tprod_fast((a.t1, a.t2), (b.t1, b.t2))
            assert np.array_equal(f1[:, rows][:, :, cols], c1) and np.array_equal(f2[:, rows][:, :, cols], c2)
            n1, n2 = O.ref_tprod_naive((a.t1, a.t2), (b.t1, b.t2))
            cfg_out["cfg1_full_fast1"], cfg_out["cfg1_full_fast2"] = f1, f2
            cfg_out["cfg1_naive_err"] = np.array(O.rel_frob_error((f1, f2), (n1, n2)))
        print(f"cfg{c}: {len(rows)} rows x {len(cols)} cols sampled", flush=True)
    np.savez_compressed(os.path.join(HERE, "configs.npz"), **cfg_out)

    # a QT3 file written by the reference's own write_tensor (tensor_io.cpp:85-92)
    O.ref_write_tensor(os.path.join(HERE, "ref_gen_3x2x4_seed9.qt3"), O.ref_gen_random_tensor(3, 2, 4, 9))


if __name__ == "__main__":
    main()
