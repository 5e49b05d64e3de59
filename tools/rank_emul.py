"""Time one rank's share of the row-sharded pipeline on one GPU (all B chunks
loaded locally, no broadcast): the per-rank compute of bench.py under torchrun."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2212_14318_b200 as qt
from paper_2212_14318_b200.configs import CONFIGS
from paper_2212_14318_b200.distributed import FreqParallelTProduct, Grid2DTProduct, RowShardedTProduct
cfg = CONFIGS[int(os.environ.get("CFG", 5))]
a, b = qt.make_inputs(cfg)
for world in [int(w) for w in os.environ.get("WORLDS", "1,2,4,8").split(",")]:
    if os.environ.get("MODE", "grid") == "freq":
        # rank 0's stages (K1 of its rows, stage 2 of its slots, K3 of its rows);
        # the exchanged pieces are replaced by finite random data
        sh = FreqParallelTProduct(cfg.m, cfg.n, cfg.s, cfg.p, 0, world, "cuda:0")
        sh.load_a(a.t1, a.t2)
        sh.load_b(b.t1, b.t2)
        for t in (sh.ac, sh.bc):
            t.normal_()

        def one():
            sh.k1()
            sh.k2_multiply(sh.k2_prepare())
            sh.k3()
        sh.step = one
        xfer = sum(v.numel() * 8 for v, peer in sh.sends_a() + sh.sends_b() + sh.sends_c() if peer != 0)
        print(f"world {world}: rank 0 sends {xfer / 1e9:.2f} GB per step (and receives about as much)")
    elif os.environ.get("MODE", "grid") == "rows":
        sh = RowShardedTProduct(cfg.m, cfg.n, cfg.s, cfg.p, 0, world, "cuda:0", nchunks=int(os.environ.get("NCH", 8)))
        sh.load_a(a.t1, a.t2)
    else:
        sh = Grid2DTProduct(cfg.m, cfg.n, cfg.s, cfg.p, 0, world, "cuda:0")
        sh.load_a(a.t1, a.t2, owned_only=False)
    if not hasattr(sh, "ns"):
        sh.load_b(b.t1, b.t2, owned_only=False)
    for _ in range(2):
        sh.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        sh.step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    grid = (f" grid {sh.gr}x{sh.gc} block {sh.rows}x{sh.cols}" if hasattr(sh, "gr") else
            f" slots [{sh.s0}, {sh.s1})" if hasattr(sh, "ns") else f" {sh.rows} rows")
    print(f"world {world}:{grid}: rank 0 {ms:.2f} ms/step; ideal {67.3 / world:.2f}; eff {67.3 / world / ms:.2f}",
          flush=True)
    del sh
    torch.cuda.empty_cache()
