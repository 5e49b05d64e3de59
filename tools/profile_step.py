#!/usr/bin/env python3
"""One device-resident T-product step for profilers (ncu launch lists and
--set full captures): W warm-up steps then K steps of the product pipeline
K1 -> K2 -> K3 on a BASELINE config, nothing else on the GPU."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2212_14318_b200 as qt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=1)
args = ap.parse_args()
cfg = qt.CONFIGS[args.config]
a, b = qt.make_inputs(cfg)
dev = torch.device("cuda", 0)
t = {k: torch.from_numpy(v.view(np.float64)).to(dev) for k, v in
     (("a1", a.t1), ("a2", a.t2), ("b1", b.t1), ("b2", b.t2))}
c1 = torch.empty((cfg.p, cfg.m, 2 * cfg.s), dtype=torch.float64, device=dev)
c2 = torch.empty_like(c1)
for i in range(args.warmup + args.steps):
    qt.tprod_fast_device(t["a1"], t["a2"], t["b1"], t["b2"], c1, c2, cfg.m, cfg.n, cfg.s, cfg.p)
torch.cuda.synchronize()
print("ok", cfg.name, float(c1.abs().sum()))
