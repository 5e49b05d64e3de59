"""Launch timeline of one T-product step (qt_prof_enable(2)): every tagged
kernel's start/end on its stream, ms from the step start.  CFG=5 by default."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2212_14318_b200 as qt
from paper_2212_14318_b200.configs import CONFIGS

cfg = CONFIGS[int(os.environ.get("CFG", 5))]
L = qt._native.lib()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(1)
a1, a2 = (torch.randn((cfg.p, cfg.m, 2 * cfg.n), dtype=torch.float64, device=dev, generator=g) for _ in range(2))
b1, b2 = (torch.randn((cfg.p, cfg.n, 2 * cfg.s), dtype=torch.float64, device=dev, generator=g) for _ in range(2))
c1, c2 = (torch.empty((cfg.p, cfg.m, 2 * cfg.s), dtype=torch.float64, device=dev) for _ in range(2))


def step():
    qt._native.check(L.qt_tprod_f64_device(a1.data_ptr(), a2.data_ptr(), b1.data_ptr(), b2.data_ptr(), c1.data_ptr(),
                                           c2.data_ptr(), cfg.m, cfg.n, cfg.s, cfg.p, None), "tprod")


for _ in range(3):
    step()
torch.cuda.synchronize()
L.qt_prof_enable(2)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
step()
e1.record()
torch.cuda.synchronize()
L.qt_prof_enable(0)
buf = ctypes.create_string_buffer(1 << 20)
n = L.qt_prof_timeline(buf, len(buf))
lines = [ln.split() for ln in buf.value.decode().splitlines()]
streams = {}
rows = []
for tag, st, t0, t1 in lines:
    streams.setdefault(st, len(streams))
    rows.append((float(t0), float(t1), tag, streams[st]))
rows.sort()
base = rows[0][0] if rows else 0.0
tot = {}
for t0, t1, tag, si in rows:
    tot[tag] = tot.get(tag, 0.0) + t1 - t0
print(f"step {e0.elapsed_time(e1):.2f} ms (events around the call); {len(rows)} tagged launches; "
      + ", ".join(f"{k} {v:.2f}" for k, v in sorted(tot.items())), flush=True)
for t0, t1, tag, si in ([] if os.environ.get("QUIET") else rows):
    print(f"  s{si} {t0 - base:8.3f} {t1 - base:8.3f} {t1 - t0:7.3f}  {tag}")
