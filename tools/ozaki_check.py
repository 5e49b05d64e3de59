"""Ozaki (int8 tcgen05) K2 vs the DMMA K2 and the oracle.  Run twice:
QTB_OZAKI=2 python tools/ozaki_check.py save oz ; QTB_OZAKI=0 ... save dm ; ... compare."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_14318_b200 as qt  # noqa: E402

SHAPES = [(24, 16, 20, 6), (64, 96, 80, 8), (130, 256, 70, 16), (1, 32, 1, 5), (200, 48, 300, 7),
          (256, 256, 256, 64), (129, 272, 131, 3)]
OUT = "/tmp/ozcheck"
if os.environ.get("OZC_SHAPES"):
    SHAPES = [tuple(int(v) for v in t.split(",")) for t in os.environ["OZC_SHAPES"].split(";")]


def main():
    mode, tag = sys.argv[1], sys.argv[2]
    os.makedirs(OUT, exist_ok=True)
    if mode == "save":
        for (m, n, s, p) in SHAPES:
            a = qt.gen_random_tensor(m, n, p, 11 + m)
            b = qt.gen_random_tensor(n, s, p, 12 + s)
            t0 = time.time()
            c = qt.tprod_fast(a, b)
            dt = time.time() - t0
            np.savez(os.path.join(OUT, f"{tag}_{m}_{n}_{s}_{p}.npz"), t1=c.t1, t2=c.t2)
            print(tag, (m, n, s, p), f"{dt*1e3:.1f} ms", flush=True)
    else:
        import oracle as O
        for (m, n, s, p) in SHAPES:
            oz = np.load(os.path.join(OUT, f"oz_{m}_{n}_{s}_{p}.npz"))
            dm = np.load(os.path.join(OUT, f"dm_{m}_{n}_{s}_{p}.npz"))
            e = O.rel_frob_error((oz["t1"], oz["t2"]), (dm["t1"], dm["t2"]))
            msg = f"{(m, n, s, p)} oz vs dmma {e:.3e}"
            if m * n * s * p <= 2e6:
                a = O.gen_random_tensor(m, n, p, 11 + m)
                b = O.gen_random_tensor(n, s, p, 12 + s)
                ref = O.tprod_fast(a, b)
                nv = O.tprod_naive(a, b)
                msg += (f" | vs ref: oz {O.rel_frob_error((oz['t1'], oz['t2']), ref):.3e} "
                        f"dm {O.rel_frob_error((dm['t1'], dm['t2']), ref):.3e} | vs naive: "
                        f"oz {O.rel_frob_error((oz['t1'], oz['t2']), nv):.3e} "
                        f"dm {O.rel_frob_error((dm['t1'], dm['t2']), nv):.3e} ref {O.rel_frob_error(ref, nv):.3e}")
            print(msg, flush=True)


if __name__ == "__main__":
    main()
