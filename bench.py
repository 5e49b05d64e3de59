#!/usr/bin/env python3
"""bench.py — T-product throughput (effective fp64 GFLOP/s) on B200.

Workload: BASELINE.json configs[4], the 1/2/4/8-GPU scaling case
(m = n = s = 2048, p = 32, components U[-1,1) from the reference generator),
override with --config {1..5}.  One step = one full T-product C = A *_T B
(K1 tube FFT of A and B -> K2 paired-frequency GEMM -> K3 inverse tube FFT)
over inputs already resident in HBM.  K2 runs as the exact int8 tcgen05
product (Ozaki-II, csrc/qt_ozaki.cu) for wide products (configs 5 and larger)
and on the fp64 DMMA tensor cores otherwise (qt_gemm_algo).  With N ranks
(torchrun, one process per GPU) the library's per-rank driver (csrc/qt_rank.cu,
its own NCCL communicator) runs the step: --multi rows = the north_star split
(rows of A and C in slabs, B broadcast once inside the timed step), --multi
freq = frequency-parallel (NCCL send/recv of the transformed pieces inside
the timed step, nothing replicated; the default for int8 products).  Strong
scaling: total work fixed.

metric value = F_eff / step time, F_eff = 32 m n s p + 10 (mn + ns + ms) p log2 p
(SURVEY §8(d)).  e2e = the same metric through the host-buffer C-ABI call
qt_tprod_f64_host (pinned host in/out, H2D + D2H inside the timed region).

--impl reference times the reference's own CPU tprod_fast (oracle/_ref, built
from /root/reference's sources) on the host cores over bounded tiles of the
same workload.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

def load_own_peaks():
    """The tensor-pipe peaks this repo measured on the B200 pool
    (profiles/r02/peaks.json: tools/microbench/int8_peak.cu and fp64_peak.cu,
    burst and sustained) — MEASURED_PEAKS.json has HBM and bf16 only."""
    with open(os.path.join(ROOT, "profiles", "r02", "peaks.json")) as f:
        return json.load(f)


OWN_PEAKS = load_own_peaks()
# fp64 DMMA: burst and sustained agree (37.16 / 37.15 TF/s, no power cap at 781 W)
PEAK_FP64_DMMA_TFLOPS = OWN_PEAKS["fp64_dmma_tflops"]["sustained"]


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def ncu_traffic(cfg, kernel: str, rows: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the latest committed ncu capture of this config (profiles/r*/ncu_traffic_cfgN.json),
    only when this run's launch is the captured one (full rows, N = 1)."""
    import glob
    if rows != cfg.m:
        return None, None
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", f"ncu_traffic_cfg{cfg.idx}.json")))
    if not files:
        return None, None
    with open(files[-1]) as f:
        d = json.load(f)
    rec = d.get("per_launch", {}).get(kernel)
    if not rec:
        return None, None
    return rec.get("traffic_bytes"), os.path.relpath(files[-1], ROOT)


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-tile", type=int, default=0, help="reference tile edge (0 = auto)")
    ap.add_argument("--multi", choices=["auto", "rows", "freq"], default="auto",
                    help="N > 1 decomposition (csrc/qt_rank.cu): rows = the north_star split (rows of A and C in "
                         "slabs, B broadcast once with NCCL); freq = frequency-parallel (rows of A/B/C for the "
                         "tube FFTs, frequency slots for stage 2, NCCL send/recv of the pieces, nothing "
                         "replicated); auto = freq when the product takes the int8 stage 2, else rows")
    ap.add_argument("--exchange", choices=["nccl", "fused"], default="nccl",
                    help="frequency-parallel exchange: nccl = send/recv groups; fused = K1 stores / K3 loads "
                         "straight into / from the peers' stage buffers (CUDA IPC over NVLink, the library's "
                         "device barrier; not yet run on more than one GPU)")
    ap.add_argument("--sharded", action="store_true",
                    help="run the N > 1 per-rank driver even on one GPU (a one-rank NCCL communicator)")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle sampling DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self._t.join(timeout=2)

    def summary(self):
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = max(smax, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------- CPU reference
def reference_tiles(cfg, tile: int, count: int, seed: int = 7):
    """`count` (row-slab x column-slab) tiles of the workload, spread over C."""
    rng = np.random.default_rng(seed)
    tr, tc = min(tile, cfg.m), min(tile, cfg.s)
    nr, nc = -(-cfg.m // tr), -(-cfg.s // tc)
    picks = rng.choice(nr * nc, size=min(count, nr * nc), replace=False)
    out = []
    for k in picks:
        r0, c0 = (int(k) // nc) * tr, (int(k) % nc) * tc
        out.append((r0, min(cfg.m, r0 + tr), c0, min(cfg.s, c0 + tc)))
    return out, nr * nc


def time_reference(cfg, a, b, tile: int, threads: int):
    """Run the UNMODIFIED reference tprod_fast (oracle/_ref) on `threads`
    tiles in parallel, one host thread each (ctypes releases the GIL).  Each
    tile is bitwise the matching block of the reference's full result (rows
    of C depend only on rows of A, columns only on columns of B), so
    (tile fraction of F_eff) / wall time is the reference's throughput on the
    workload with `threads` host cores busy.  a, b: (t1, t2) host planes."""
    import oracle as O
    tiles, total = reference_tiles(cfg, tile, threads)
    jobs = []
    for (r0, r1, c0, c1) in tiles:
        at = (np.ascontiguousarray(a[0][:, r0:r1, :]), np.ascontiguousarray(a[1][:, r0:r1, :]))
        bt = (np.ascontiguousarray(b[0][:, :, c0:c1]), np.ascontiguousarray(b[1][:, :, c0:c1]))
        jobs.append((at, bt))
    th = [threading.Thread(target=O.ref_tprod_fast, args=j) for j in jobs]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    wall = time.perf_counter() - t0
    frac = sum((r1 - r0) * (c1 - c0) for (r0, r1, c0, c1) in tiles) / float(cfg.m * cfg.s)
    gflops = frac * cfg.flops_eff / wall / 1e9
    sample = (f"{len(tiles)} tile(s) of {tiles[0][1] - tiles[0][0]} rows x {tiles[0][3] - tiles[0][2]} cols "
              f"({frac * 100:.3f}% of C), one tile per thread, reference tprod_fast unmodified")
    return gflops, wall, sample, len(tiles)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_reference(cfg, a, b, tile: int, threads: int):
    """The reference's CPU path on this host: all cores (tile-parallel) and
    one core (one tile, one thread), plus the CPU model."""
    g, w, sample, used = time_reference(cfg, a, b, tile, threads)
    g1, w1, sample1, _ = time_reference(cfg, a, b, tile, 1)
    return {"value": g, "unit": "GFLOP/s", "cores": used, "kind": "reference", "sample": sample, "wall_s": w,
            "cpu_model": cpu_model(), "nproc": os.cpu_count(),
            "single_core": {"value": g1, "unit": "GFLOP/s", "cores": 1, "sample": sample1, "wall_s": w1}}


def load_configs():
    """The BASELINE config table (paper_2212_14318_b200/configs.py) loaded by
    path: standalone, so the reference arm never imports the product package
    or loads its library."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("qt_bench_configs",
                                                  os.path.join(ROOT, "paper_2212_14318_b200", "configs.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod  # (dataclasses resolve annotations through sys.modules)
    spec.loader.exec_module(mod)
    return mod.CONFIGS


def config_dict(cfg):
    """The `config` object of both arms' JSON lines (identical by construction)."""
    return {"workload": cfg.name, "m": cfg.m, "n": cfg.n, "s": cfg.s, "p": cfg.p}


def auto_tile(cfg):
    # ~10-25 s of single-thread reference work per tile on a ~3 GHz Xeon
    return {1: 8, 2: 128, 3: 16, 4: 64, 5: 128}.get(cfg.idx, 64)


def host_inputs(cfg, pinned: bool, need_b: bool = True):
    """Seeded host inputs (reference generator / SURVEY §8(d) distributions).
    B is skipped (None) when need_b is False (ranks != 0 of a sharded run)."""
    import torch

    import paper_2212_14318_b200 as qt
    sa, sb = cfg.seeds()

    def alloc(rows, cols):
        t = torch.empty((cfg.p, rows, cols, 2), dtype=torch.float64, pin_memory=pinned)
        return t, t.numpy().view(np.complex128)[..., 0]

    bufs = {}
    bufs["a1"], v1 = alloc(cfg.m, cfg.n)
    bufs["a2"], v2 = alloc(cfg.m, cfg.n)
    # CdTensor3 keeps views of the (pinned) buffers (no copy): generate in place
    a = qt.CdTensor3(cfg.m, cfg.n, cfg.p, v1, v2)
    assert a.t1.ctypes.data == bufs["a1"].data_ptr()
    qt.gen_tensor(cfg.m, cfg.n, cfg.p, sa, cfg.dist_a, cfg.scale_a, out=a)
    b = None
    if need_b:
        bufs["b1"], w1 = alloc(cfg.n, cfg.s)
        bufs["b2"], w2 = alloc(cfg.n, cfg.s)
        b = qt.CdTensor3(cfg.n, cfg.s, cfg.p, w1, w2)
        qt.gen_tensor(cfg.n, cfg.s, cfg.p, sb, cfg.dist_b, cfg.scale_b, out=b)
    return a, b, bufs


def run_reference(args, cfg):
    """The reference's own CPU tprod_fast (oracle/_ref, compiled from
    /root/reference's sources, unmodified) on this host's cores.  Inputs come
    from the oracle's generators (the reference's gen_random_tensor and the
    restated normal / pure-quaternion ones) — this arm imports neither the
    product package nor its library."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle as O
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libqtref.so not built "
                          "(make -C oracle ref needs /root/reference)"}))
        return 0
    sa, sb = cfg.seeds()
    a = O.gen_tensor(cfg.dist_a, cfg.m, cfg.n, cfg.p, sa, cfg.scale_a)
    b = O.gen_tensor(cfg.dist_b, cfg.n, cfg.s, cfg.p, sb, cfg.scale_b)
    threads = os.cpu_count() or 1
    tile = args.cpu_tile or auto_tile(cfg)
    for _ in range(args.warmup):
        time_reference(cfg, a, b, max(8, tile // 4), threads)
    vals, walls = [], []
    for _ in range(args.steps):
        g, w, sample, used = time_reference(cfg, a, b, tile, threads)
        vals.append(g)
        walls.append(w)
    value = statistics.median(vals)
    g1, w1, sample1, _ = time_reference(cfg, a, b, tile, 1)
    line = {
        "impl": "reference",
        "metric": "T-product throughput (effective fp64 GFLOP/s)",
        "value": value, "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(walls) * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded; reference generator / SURVEY §8d distributions)",
        "config": config_dict(cfg),
        "parallelism": f"{used} host threads, tile-parallel (one (row x column) tile of C per thread)",
        "flops_eff_per_step": cfg.flops_eff,
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": used, "kind": "reference", "sample": sample,
                         "cpu_model": cpu_model(), "nproc": os.cpu_count(),
                         "single_core": {"value": g1, "unit": "GFLOP/s", "cores": 1, "sample": sample1,
                                         "wall_s": w1}},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------- our arm
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2212_14318_b200 as qt
    from paper_2212_14318_b200 import shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    L = qt._native.lib()
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream

    lo, hi = shard.row_slab(cfg.m, world, rank)
    rows, cols = hi - lo, cfg.s  # this rank's block of C (whole C at N = 1)
    mode = "rows"
    k2_shape = None  # (rows, cols, frequencies) of this rank's stage 2, if not (rows, cols, p)
    # N = 1: pinned host inputs (the e2e leg copies from them); N > 1: every
    # rank regenerates A and B (sequential generator) and keeps the pieces it owns
    sharded_mode = world > 1 or args.sharded
    a, b, _ = host_inputs(cfg, pinned=not sharded_mode, need_b=True)
    # L2 flush between timed steps of products smaller than L2: write a 256 MB
    # buffer (> 126 MB L2), then read another one, so the L2 holds neither the
    # inputs nor dirty lines whose write-back would land inside the next timed
    # step (126 MB of write-back is ~19 us of HBM time)
    l2_buf = torch.zeros(2, 64 * 1024 * 1024, dtype=torch.float32, device=dev)

    def l2_flush_now():
        l2_buf[0].zero_()
        l2_buf[1].sum()
    big = (cfg.bytes_tensor(rows, cfg.n) + cfg.bytes_tensor(cfg.n, cfg.s)) > 2 * 126e6
    if not sharded_mode:
        # device-resident inputs; one step = the product entry point qt_tprod_f64_device
        da1 = torch.from_numpy(a.t1.view(np.float64)).to(dev)
        da2 = torch.from_numpy(a.t2.view(np.float64)).to(dev)
        db1 = torch.from_numpy(b.t1.view(np.float64)).to(dev)
        db2 = torch.from_numpy(b.t2.view(np.float64)).to(dev)
        dc1 = torch.empty((cfg.p, rows, 2 * cfg.s), dtype=torch.float64, device=dev)
        dc2 = torch.empty_like(dc1)

        def step():
            rc = L.qt_tprod_f64_device(da1.data_ptr(), da2.data_ptr(), db1.data_ptr(), db2.data_ptr(),
                                       dc1.data_ptr(), dc2.data_ptr(), rows, cfg.n, cfg.s, cfg.p, sh)
            qt._native.check(rc, "tprod_fast")
    else:
        # one process per GPU: the library's per-rank driver (csrc/qt_rank.cu)
        # owns the NCCL communicator and every transfer; each rank keeps only
        # its inputs (its rows of A, and B on the root / its rows of B)
        from paper_2212_14318_b200 import distributed
        mode = args.multi
        if mode == "auto":
            mode = "freq" if L.qt_gemm_algo(cfg.m, cfg.n, cfg.s, cfg.p) == 1 else "rows"
        comm = distributed.RankComm(rank, world, local, dist if world > 1 else None)
        cls = distributed.FreqTProduct if mode == "freq" else distributed.RowsTProduct
        sharded = cls(comm, cfg.m, cfg.n, cfg.s, cfg.p)
        if mode == "freq" and args.exchange == "fused":
            handles = [None] * world
            if world > 1:
                dist.all_gather_object(handles, sharded.ipc_handle())
            else:
                handles = [sharded.ipc_handle()]
            sharded.set_peers(handles)
        sharded.load_a(a.t1, a.t2)
        sharded.load_b(b.t1, b.t2)
        pin_own = []  # (device buffer, pinned host copy) this rank uploads on the e2e leg
        for t in sharded.owned():
            pt = torch.empty(t.shape, dtype=torch.float64, pin_memory=True)
            pt.copy_(t)
            pin_own.append((t, pt))
        rows, cols = sharded.rows, cfg.s
        if world > 1:
            dist.barrier()

        def step():
            sharded.step()
        del a, b
        # stage-timing operands of this rank's block shape
        da1 = torch.randn((cfg.p, rows, 2 * cfg.n), dtype=torch.float64, device=dev)
        da2 = torch.randn_like(da1)
        db1 = torch.randn((cfg.p, cfg.n, 2 * cols), dtype=torch.float64, device=dev)
        db2 = torch.randn_like(db1)
        dc1, dc2 = sharded.c[0], sharded.c[1]
        if mode == "freq":  # this rank's stage 2: all m x s of its frequency slots
            k2_shape = (cfg.m, cfg.s, max(1, sharded.slot1 - sharded.slot0))

    # clocks are sampled from the first warm-up step through the per-kernel
    # timing loops, so short steps still yield samples under load
    clk = ClockSampler(local).__enter__()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = L.qt_kernel_launches()
    for i in range(args.steps):
        if not big:
            l2_flush_now()
        starts[i].record(stream)
        step()
        ends[i].record(stream)
    torch.cuda.synchronize()
    launches = L.qt_kernel_launches() - launches0
    if world > 1:
        tl = torch.tensor([launches], device=dev, dtype=torch.int64)
        dist.all_reduce(tl)  # every rank's kernels
        launches = int(tl.item())
        dist.barrier()
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends)) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = cfg.flops_eff / (ms * 1e-3) / 1e9  # whole-job GFLOP/s (all ranks' rows)

    # ---- per-kernel timing for the roofline (same stream, CUDA events) ----
    # (full-B stage kernels; with N > 1 ranks this rank's block / slot shape)
    krows, kcols, kp = k2_shape or (rows, cols, cfg.p)
    ah = torch.empty((2, kp, krows, 2 * cfg.n), dtype=torch.float64, device=dev)
    bh = torch.empty((2, kp, cfg.n, 2 * kcols), dtype=torch.float64, device=dev)
    kc = torch.empty((2, kp, krows, 2 * kcols), dtype=torch.float64, device=dev) if k2_shape else None
    kc1, kc2 = (kc[0], kc[1]) if k2_shape else (dc1, dc2)
    ka1 = torch.randn((kp, krows, 2 * cfg.n), dtype=torch.float64, device=dev) if k2_shape else da1
    ka2 = torch.randn_like(ka1) if k2_shape else da2
    kb1 = torch.randn((kp, cfg.n, 2 * kcols), dtype=torch.float64, device=dev) if k2_shape else db1
    kb2 = torch.randn_like(kb1) if k2_shape else db2
    qt._native.check(L.qt_qfft3_conj_f64_device(ka1.data_ptr(), ka2.data_ptr(), ah[0].data_ptr(), ah[1].data_ptr(),
                                                krows, cfg.n, kp, sh), "qfft3")
    qt._native.check(L.qt_qfft3_conj_f64_device(kb1.data_ptr(), kb2.data_ptr(), bh[0].data_ptr(), bh[1].data_ptr(),
                                                cfg.n, kcols, kp, sh), "qfft3")
    del ka1, ka2, kb1, kb2

    def timed(fn, reps):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for s0, e0 in evs:
            if not big:
                l2_flush_now()
            s0.record(stream)
            fn()
            e0.record(stream)
        torch.cuda.synchronize()
        return sum(s0.elapsed_time(e0) for s0, e0 in evs) / reps

    algo = L.qt_gemm_algo(cfg.m, cfg.n, cfg.s, cfg.p)   # 0 = fp64 DMMA, 1 = exact int8 (tcgen05)
    gemm_ms = timed(lambda: L.qt_spectral_product_f64_device_ld_algo(
        ah[0].data_ptr(), ah[1].data_ptr(), bh[0].data_ptr(), bh[1].data_ptr(), kc1.data_ptr(), kc2.data_ptr(), krows,
        cfg.n, kcols, kp, kcols, kcols, cfg.n * kcols, krows * kcols, algo, sh), max(2, args.steps))
    # stage-2 accuracy of the algorithm this workload takes, on this run's data:
    # the int8 (exact modular) result against the fp64 DMMA result (both on the GPU)
    accuracy = None
    if algo == 1:
        c8 = torch.empty((2, kp, krows, 2 * kcols), dtype=torch.float64, device=dev)
        cd = torch.empty_like(c8)
        for algo_id, dst in ((1, c8), (0, cd)):
            qt._native.check(L.qt_spectral_product_f64_device_ld_algo(
                ah[0].data_ptr(), ah[1].data_ptr(), bh[0].data_ptr(), bh[1].data_ptr(), dst[0].data_ptr(),
                dst[1].data_ptr(), krows, cfg.n, kcols, kp, kcols, kcols, cfg.n * kcols, krows * kcols, algo_id, sh),
                "spectral(accuracy)")
        torch.cuda.synchronize()
        num = float(torch.linalg.vector_norm(c8 - cd).item())
        den = float(torch.linalg.vector_norm(cd).item())
        accuracy = {"k2_int8_vs_fp64_dmma_rel_frob": num / den if den else 0.0,
                    "note": "stage 2 of this step's operands evaluated both ways on the GPU; the int8 path is "
                            "exact in integers (53-bit scaled inputs, one final rounding), tests/test_gpu_int8.py "
                            "shows its error vs a long-double truth is <= the fp64 GEMM's"}
        del c8, cd
    del ah, bh, kc
    ah = torch.empty((2, cfg.p, rows, 2 * cfg.n), dtype=torch.float64, device=dev)
    fftA_ms = timed(lambda: L.qt_qfft3_conj_f64_device(da1.data_ptr(), da2.data_ptr(), ah[0].data_ptr(),
                                                       ah[1].data_ptr(), rows, cfg.n, cfg.p, sh), max(3, args.steps))
    ifft_ms = timed(lambda: L.qt_qifft3_conj_f64_device(dc1.data_ptr(), dc2.data_ptr(), dc1.data_ptr(),
                                                        dc2.data_ptr(), rows, cols, cfg.p, sh), max(3, args.steps))
    del ah
    # ---- per-kernel device time of the stage-2 GEMM kernel itself (library
    # CUDA events on the launching stream, qt_prof_*), over a few extra steps
    nprof = max(2, args.steps)
    L.qt_prof_enable(1)
    for _ in range(nprof):
        if not big:
            l2_flush_now()
        step()
    torch.cuda.synchronize()
    L.qt_prof_enable(0)
    def read_prof(steps_done=None):
        steps_done = steps_done or nprof
        out = {}
        for tag in ("small_fused", "fft", "k2_dmma", "k2_int8_gemm", "k2_int8_residues", "k2_int8_residues_b", "k2_int8_colnorms",
                    "k2_int8_crt"):
            t_ms, n_l = ctypes.c_double(0.0), ctypes.c_uint64(0)
            qt._native.check(L.qt_prof_read(tag.encode(), ctypes.byref(t_ms), ctypes.byref(n_l)), "qt_prof_read")
            if n_l.value:
                out[tag] = {"ms_per_step": t_ms.value / steps_done, "launches_per_step": n_l.value / steps_done}
        return out

    prof = read_prof()
    # the int8 GEMM alone on the SMs (frequency batches in order, no co-running
    # residue/CRT kernels): the kernel's own rate, reported beside the live one
    prof_iso = {}
    if algo == 1:
        old_pipe = os.environ.get("QTB_OZAKI_PIPE")
        os.environ["QTB_OZAKI_PIPE"] = "0"
        L.qt_prof_enable(1)
        for _ in range(nprof):
            step()
        torch.cuda.synchronize()
        L.qt_prof_enable(0)
        prof_iso = read_prof()
        if old_pipe is None:
            del os.environ["QTB_OZAKI_PIPE"]
        else:
            os.environ["QTB_OZAKI_PIPE"] = old_pipe
    # keep the GPU under the same load for >= 1 s of clock samples
    # (iteration count from the max-over-ranks step time: identical on every rank)
    for _ in range(min(2000, int(math.ceil(1000.0 / max(ms, 1e-3))))):
        step()
    torch.cuda.synchronize()
    clk.__exit__(None, None, None)
    peaks, peak_src = load_peaks()
    gauss = os.environ.get("QTB_GEMM", "3m")[:1] != "4"
    gemm_tf = 32.0 * krows * cfg.n * kcols * kp / (gemm_ms * 1e-3) / 1e12   # algorithmic (reference) flops
    exec_tf = gemm_tf * (0.75 if gauss else 1.0)                              # DMMA flops actually executed
    fftA_gbs = 2 * cfg.bytes_tensor(rows, cfg.n) / (fftA_ms * 1e-3) / 1e9
    ifft_gbs = 2 * cfg.bytes_tensor(rows, cols) / (ifft_ms * 1e-3) / 1e9
    gemm_bytes = (cfg.bytes_tensor(krows, cfg.n) + cfg.bytes_tensor(cfg.n, kcols) + cfg.bytes_tensor(krows, kcols)) \
        * kp / cfg.p
    gemm_ai = 32.0 * krows * cfg.n * kcols * kp / gemm_bytes
    ridge = PEAK_FP64_DMMA_TFLOPS * 1e12 / (peaks["hbm_gbs"] * 1e9)
    # the DMMA stage-2 kernel this shape takes (qt_gemm.cu dmma_impl)
    k2_name = ("K2 paired_tiny_ws_kernel (warp-specialised: bulk-copy producer warp, mbarrier ring; DMMA.8x8x4)"
               if gauss and krows <= 16 and kcols <= 16 and cfg.n <= 16 else "K2 paired_spectral_gemm (DMMA.8x8x4)")
    algo_txt = ("gauss-3m: each complex product as 3 real DMMA products (24 m n s p executed flops)" if gauss
                else "4m: each complex product as 4 real DMMA products (32 m n s p executed flops)")
    if algo == 1 and "k2_int8_gemm" in prof:
        # exact int8 path: 15 modular GEMMs of the real-embedded (2m x 4n) . (4n x 2s) product per frequency
        k_ms = prof["k2_int8_gemm"]["ms_per_step"]
        ops = 2.0 * 15 * (2 * krows) * (4 * cfg.n) * (2 * kcols) * kp
        ach = ops / (k_ms * 1e-3) / 1e12
        # the GEMM runs ~50 ms inside a long power-capped step: the sustained
        # tcgen05 int8 rate is its ceiling (burst reported beside it)
        peak_i8 = OWN_PEAKS["int8_tcgen05_tops"]["sustained"]
        peak_i8_burst = OWN_PEAKS["int8_tcgen05_tops"]["burst"]
        roof = {"kernel": "K2 int8 modular GEMM oz_gemm2_kernel (tcgen05.mma.cta_group::2.kind::i8, TMA, TMEM)",
                "bound": "tensor", "achieved": ach, "peak": peak_i8, "unit": "TFLOP/s", "frac": ach / peak_i8,
                "op_type": "int8 x int8 -> int32 tensor ops (multiply-add = 2), i.e. TOPS",
                "peak_source": "measured tcgen05 kind::i8 throughput, sustained (back-to-back 4 s under the "
                               "power cap, 1612 MHz): profiles/r02/peaks.json (tools/microbench/int8_peak.cu)",
                "peak_burst": peak_i8_burst, "frac_of_burst": ach / peak_i8_burst,
                "frac_of_2x_measured_bf16_sustained": (ach / (2.0 * peaks["bf16_tflops_sustained"])
                                                       if "bf16_tflops_sustained" in peaks else None),
                "algorithmic": "2 * 15 moduli * (2m)(4n)(2s) * p int8 ops per step (= 480 m n s p), "
                               "launched in frequency batches",
                "algorithm": "exact Ozaki-II: 53-bit scaled integers (norm-bounded), 15 coprime moduli <= 256, CRT (csrc/qt_ozaki.cu)",
                "kernel_ms": k_ms, "launches_per_step": prof["k2_int8_gemm"]["launches_per_step"],
                "share_of_step": k_ms / ms,
                "fp64_equivalent_tflops": 32.0 * krows * cfg.n * kcols * kp / (k_ms * 1e-3) / 1e12,
                "concurrency": "frequency batches software-pipelined over two streams: the residue and CRT "
                               "kernels of neighbouring batches run beside this kernel (kernel_ms is its own "
                               "event-timed duration, which includes that sharing)",
                "traffic": None}
        # the same rate against the peak at the SM clock this run held (the
        # power cap sets the clock; the rated burst is 4387 TOPS at 1965 MHz)
        csum = clk.summary()
        if csum.get("sm_mhz"):
            per_clk = peak_i8_burst / 1965.0 * csum["sm_mhz"]
            roof["frac_at_measured_clock"] = ach / per_clk
            roof["peak_at_measured_clock"] = per_clk
        if "k2_int8_gemm" in prof_iso:
            iso_ms = prof_iso["k2_int8_gemm"]["ms_per_step"]
            roof["isolated"] = {"kernel_ms": iso_ms, "achieved": ops / (iso_ms * 1e-3) / 1e12,
                                "frac": ops / (iso_ms * 1e-3) / 1e12 / peak_i8,
                                "note": "same kernel, batches in order (QTB_OZAKI_PIPE=0), nothing co-running"}
        traffic, traffic_src = ncu_traffic(cfg, "K2_int8_gemm", rows if k2_shape is None else -1)
        roof["algorithmic_bytes"] = None
    elif "small_fused" in prof:
        # the whole product is ONE cluster kernel (csrc/qt_small.cu): A and B
        # read once, C written once, K1 -> K2 -> K3 exchanged through DSMEM
        k_ms = prof["small_fused"]["ms_per_step"]
        fused_bytes = cfg.bytes_tensor(rows, cfg.n) + cfg.bytes_tensor(cfg.n, cols) + cfg.bytes_tensor(rows, cols)
        gb = fused_bytes / (k_ms * 1e-3) / 1e9
        roof = {"kernel": "one-launch small product small_tprod_kernel (K1 + K2 + K3 in one thread-block-cluster "
                          "kernel, DSMEM exchanges, DMMA.8x8x4 stage 2)",
                "bound": "hbm", "achieved": gb, "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": gb / peaks["hbm_gbs"],
                "peak_source": f"{peak_src} hbm_gbs (MEASURED_PEAKS.json)",
                "algorithmic": "32*(mn+ns+ms)*p bytes per launch (A and B read once, C written once)",
                "algorithm": algo_txt, "kernel_ms": k_ms, "share_of_step": k_ms / ms,
                "latency_floor": "an EMPTY kernel timed the same way (after the 256 MB L2 flush, events on the "
                                 "stream) takes 6.1 us and a CUDA graph of three 1 MB copies 10.2 us on this "
                                 "B200 (tools/microbench/launch_probe.cu, profiles/r02/launch_probe.txt): the "
                                 "product is latency-bound, not HBM-bound",
                "traffic": None}
        traffic, traffic_src = None, None
        roof["algorithmic_bytes"] = fused_bytes
    elif gemm_ai >= ridge:
        k_ms = prof.get("k2_dmma", {}).get("ms_per_step", gemm_ms)
        ktf = 32.0 * krows * cfg.n * kcols * kp / (k_ms * 1e-3) / 1e12
        roof = {"kernel": k2_name, "bound": "tensor", "achieved": ktf,
                "peak": PEAK_FP64_DMMA_TFLOPS, "unit": "TFLOP/s", "frac": ktf / PEAK_FP64_DMMA_TFLOPS,
                "peak_source": "measured fp64 DMMA (mma.sync.m8n8k4.f64) sustained = burst, profiles/r02/peaks.json "
                               "(tools/microbench/fp64_peak.cu); MEASURED_PEAKS.json has no fp64",
                "algorithmic": "32*m*n*s*p flops per launch (SURVEY 8d F_gemm, the reference's 16 m n s p "
                               "multiplications + additions)",
                "algorithm": algo_txt, "executed_tflops": ktf * (0.75 if gauss else 1.0),
                "executed_frac": ktf * (0.75 if gauss else 1.0) / PEAK_FP64_DMMA_TFLOPS,
                "kernel_ms": k_ms, "share_of_step": k_ms / ms, "traffic": None}
        traffic, traffic_src = ncu_traffic(cfg, "K2_gemm", rows if k2_shape is None else -1)
        roof["algorithmic_bytes"] = gemm_bytes
    else:
        k_ms = prof.get("k2_dmma", {}).get("ms_per_step", gemm_ms)
        gb = gemm_bytes / (k_ms * 1e-3) / 1e9
        roof = {"kernel": k2_name, "bound": "hbm", "achieved": gb,
                "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": gb / peaks["hbm_gbs"],
                "peak_source": f"{peak_src} hbm_gbs (MEASURED_PEAKS.json)",
                "algorithmic": "32*(mn+ns+ms)*p bytes per launch", "algorithm": algo_txt,
                "kernel_ms": k_ms, "share_of_step": k_ms / ms, "traffic": None}
        traffic, traffic_src = ncu_traffic(cfg, "K2_gemm", rows if k2_shape is None else -1)
        roof["algorithmic_bytes"] = gemm_bytes
    roof["traffic"] = traffic
    roof["traffic_source"] = traffic_src
    roof["kernel_times_ms_per_step"] = {k: v["ms_per_step"] for k, v in prof.items()}
    stages = {
        "K1_fft_A": {"ms": fftA_ms, "GB_s": fftA_gbs, "frac_hbm": fftA_gbs / peaks["hbm_gbs"]},
        "K2_gemm": {"ms": gemm_ms, "TFLOP_s": gemm_tf, "frac_fp64": gemm_tf / PEAK_FP64_DMMA_TFLOPS,
                    "algorithm": "exact int8 (Ozaki-II, tcgen05)" if algo == 1 else "fp64 DMMA",
                    **({} if algo == 1 else {"executed_TFLOP_s": exec_tf})},
        "K3_ifft_C": {"ms": ifft_ms, "GB_s": ifft_gbs, "frac_hbm": ifft_gbs / peaks["hbm_gbs"]},
    }
    if "fft" in prof:  # the step's own tube-FFT launches (K1 of A and B in one launch, K3), event-timed
        fb = 2 * (cfg.bytes_tensor(rows, cfg.n) + cfg.bytes_tensor(cfg.n, cols) + cfg.bytes_tensor(rows, cols))
        f_ms = prof["fft"]["ms_per_step"]
        stages["K1_K3_in_step"] = {"ms": f_ms, "GB_s": fb / (f_ms * 1e-3) / 1e9,
                                   "frac_hbm": fb / (f_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                                   "algorithmic": "64 (mn + ns + ms) p bytes (read + write of both planes)"}

    # ---- the fp64 DMMA stage 2 on the same step (the north_star's design), when
    # this workload's default is the int8 path: K1 -> paired DMMA GEMM -> K3
    dmma_path = None
    if algo == 1 and not sharded_mode:
        ahd = torch.empty((2, cfg.p, rows, 2 * cfg.n), dtype=torch.float64, device=dev)
        bhd = torch.empty((2, cfg.p, cfg.n, 2 * cols), dtype=torch.float64, device=dev)

        def dmma_step():
            qt._native.check(L.qt_qfft3_conj_f64_device(da1.data_ptr(), da2.data_ptr(), ahd[0].data_ptr(),
                                                        ahd[1].data_ptr(), rows, cfg.n, cfg.p, sh), "qfft3")
            qt._native.check(L.qt_qfft3_conj_f64_device(db1.data_ptr(), db2.data_ptr(), bhd[0].data_ptr(),
                                                        bhd[1].data_ptr(), cfg.n, cols, cfg.p, sh), "qfft3")
            qt._native.check(L.qt_spectral_product_f64_device_ld_algo(
                ahd[0].data_ptr(), ahd[1].data_ptr(), bhd[0].data_ptr(), bhd[1].data_ptr(), dc1.data_ptr(),
                dc2.data_ptr(), rows, cfg.n, cols, cfg.p, cols, cols, cfg.n * cols, rows * cols, 0, sh), "dmma")
            qt._native.check(L.qt_qifft3_conj_f64_device(dc1.data_ptr(), dc2.data_ptr(), dc1.data_ptr(),
                                                         dc2.data_ptr(), rows, cols, cfg.p, sh), "qifft3")

        dmma_step()
        nd = max(2, min(args.steps, 3))
        L.qt_prof_enable(1)
        t_d = timed(dmma_step, nd)
        L.qt_prof_enable(0)
        pd = read_prof(nd)
        k_d = pd.get("k2_dmma", {}).get("ms_per_step", 0.0)
        ktf_d = 32.0 * rows * cfg.n * cols * cfg.p / (k_d * 1e-3) / 1e12 if k_d else None
        dmma_path = {"ms_per_step": t_d, "value": cfg.flops_eff / (t_d * 1e-3) / 1e9, "unit": "GFLOP/s",
                     "k2_kernel_ms": k_d, "k2_algorithmic_tflops": ktf_d,
                     "k2_frac_of_fp64_peak": ktf_d / PEAK_FP64_DMMA_TFLOPS if ktf_d else None,
                     "k2_executed_frac_of_dmma_pipe": (ktf_d * (0.75 if gauss else 1.0) / PEAK_FP64_DMMA_TFLOPS
                                                       if ktf_d else None),
                     "note": "same step with stage 2 on the fp64 DMMA tensor pipe (mma.sync.m8n8k4.f64, Gauss 3M): "
                             "the north_star's FP64-tensor-core design, kept as the path for configs 1-4 and as the "
                             "non-finite fallback"}
        del ahd, bhd

    # ---- end to end: host buffers in, host buffers out, copies inside the timed region ----
    e2e = None
    if not sharded_mode and args.e2e_steps > 0:
        c1p = torch.empty((cfg.p, cfg.m, 2 * cfg.s), dtype=torch.float64, pin_memory=True)
        c2p = torch.empty_like(c1p, pin_memory=True)

        def e2e_step():
            rc = L.qt_tprod_f64_host(a.t1.ctypes.data, a.t2.ctypes.data, b.t1.ctypes.data, b.t2.ctypes.data,
                                     c1p.data_ptr(), c2p.data_ptr(), cfg.m, cfg.n, cfg.s, cfg.p, local)
            qt._native.check(rc, "tprod_fast(host)")

        for _ in range(2):  # warm-up: the first calls also set up the library's pools and staging
            e2e_step()
        torch.cuda.synchronize()
        calls = []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            e2e_step()  # synchronous: returns once C is in host memory
            calls.append(time.perf_counter() - t0)
        e2e_s = float(statistics.median(calls))
        e2e = {"value": cfg.flops_eff / e2e_s / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": cfg.bytes_tensor(cfg.m, cfg.n) + cfg.bytes_tensor(cfg.n, cfg.s),
               "d2h_bytes_per_step": cfg.bytes_tensor(cfg.m, cfg.s), "ms_per_step": e2e_s * 1e3,
               "calls_ms": [round(c * 1e3, 2) for c in calls], "statistic": "median of the timed calls",
               "api": "qt_tprod_f64_host (pinned host buffers)"}
    elif sharded_mode and args.e2e_steps > 0:
        pin_c = torch.empty(sharded.c.shape, dtype=torch.float64, pin_memory=True)

        def e2e_step():  # per rank: its owned A/B pieces H2D, broadcasts + pipeline, its C block D2H
            for t, pt in pin_own:
                t.copy_(pt, non_blocking=True)
            step()
            pin_c.copy_(sharded.c, non_blocking=True)
            torch.cuda.synchronize()

        e2e_step()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        t = torch.tensor([(time.perf_counter() - t0) / args.e2e_steps], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
        e2e = {"value": cfg.flops_eff / e2e_s / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": cfg.bytes_tensor(cfg.m, cfg.n) + cfg.bytes_tensor(cfg.n, cfg.s),
               "d2h_bytes_per_step": cfg.bytes_tensor(cfg.m, cfg.s), "ms_per_step": e2e_s * 1e3,
               "api": "per rank: its pinned inputs H2D, the per-rank driver step (NCCL inside), its pinned rows "
                      "of C D2H; max over ranks"}

    cpu = None
    if rank == 0 and not sharded_mode and not args.no_cpu_baseline:
        import oracle as O
        if O.ref_available():
            cpu = cpu_reference(cfg, (a.t1, a.t2), (b.t1, b.t2), args.cpu_tile or auto_tile(cfg),
                                os.cpu_count() or 1)

    if rank == 0:
        line = {
            "metric": "T-product throughput (effective fp64 GFLOP/s)",
            "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded; reference generator / SURVEY §8d distributions)",
            "arithmetic": ("fp64 tube FFTs; stage 2 evaluated exactly in integers on the int8 tensor cores "
                           "(u8 x u8 -> s32 tcgen05 MMAs over 15 moduli, 96-bit CRT, one fp64 rounding)"
                           if L.qt_gemm_algo(cfg.m, cfg.n, cfg.s, cfg.p) == 1 else
                           "fp64 throughout (tube FFTs; stage 2 on the fp64 DMMA tensor pipe)"),
            "accuracy": accuracy,
            "fp64_dmma_path": dmma_path,
            "config": config_dict(cfg),
            "parallelism": (f"{mode}{world}" + ((" (per-rank driver qt_rank_*, " +
                                                   ("exchange fused into K1 stores / K3 loads over peer memory)"
                                                    if mode == "freq" and args.exchange == "fused" else "NCCL)"))
                                                  if sharded_mode else "")),
            "l2": "inputs > L2" if big else "L2 flushed before each timed step (256 MB write, then a 256 MB read so no "
                                            "dirty line is written back inside the step)",
            "flops_eff_per_step": cfg.flops_eff,
            "roofline": roof,
            "stages": stages,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse_args()
    cfg = load_configs()[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
