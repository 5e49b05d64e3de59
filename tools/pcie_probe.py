#!/usr/bin/env python3
"""Host<->device copy bandwidth on the GPU box (pinned), one and both directions."""
import time

import torch

N = 1 << 30  # bytes
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d = torch.empty(N, dtype=torch.uint8, device="cuda")
d2 = torch.empty(N, dtype=torch.uint8, device="cuda")
for _ in range(2):
    d.copy_(h, non_blocking=True)
    h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()


def bw(fn, nbytes, reps=5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t0) / 1e9


print("H2D GB/s", bw(lambda: d.copy_(h, non_blocking=True), N))
print("D2H GB/s", bw(lambda: h2.copy_(d2, non_blocking=True), N))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


print("H2D+D2H concurrent GB/s (sum)", bw(both, 2 * N))
