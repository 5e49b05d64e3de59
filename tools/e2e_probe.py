#!/usr/bin/env python3
"""Time qt_tprod_f64_host (pinned host buffers) on a config; QTB_TRACE=1 prints phases."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2212_14318_b200 as qt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
cfg = qt.CONFIGS[args.config]
a, b, _ = bench.host_inputs(cfg, pinned=True)
c1 = torch.empty((cfg.p, cfg.m, 2 * cfg.s), dtype=torch.float64, pin_memory=True)
c2 = torch.empty_like(c1, pin_memory=True)
L = qt._native.lib()
for r in range(args.reps + 1):
    if r == args.reps:
        os.environ["QTB_TRACE"] = "1"
    t0 = time.perf_counter()
    rc = L.qt_tprod_f64_host(a.t1.ctypes.data, a.t2.ctypes.data, b.t1.ctypes.data, b.t2.ctypes.data,
                             c1.data_ptr(), c2.data_ptr(), cfg.m, cfg.n, cfg.s, cfg.p, 0)
    qt._native.check(rc, "host")
    print(f"rep {r}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
