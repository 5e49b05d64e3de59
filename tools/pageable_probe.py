#!/usr/bin/env python3
"""Drop-in-style call on pageable host memory (numpy arrays, like std::vector):
time qt.tprod_fast vs the pinned-buffer e2e path for one config."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_14318_b200 as qt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
args = ap.parse_args()
cfg = qt.CONFIGS[args.config]
a, b = qt.make_inputs(cfg)  # pageable numpy planes
qt.tprod_fast(a, b)
for r in range(2):
    t0 = time.perf_counter()
    c = qt.tprod_fast(a, b)
    dt = time.perf_counter() - t0
    print(f"pageable tprod_fast {cfg.name}: {dt * 1e3:.1f} ms  ({cfg.flops_eff / dt / 1e12:.2f} TF/s eff)", flush=True)
