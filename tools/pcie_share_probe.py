import torch
N = 1 << 30
h = torch.empty(2 * N, dtype=torch.uint8, pin_memory=True); h2 = torch.empty(N // 2, dtype=torch.uint8, pin_memory=True)
d = torch.empty(2 * N, dtype=torch.uint8, device="cuda"); d2 = torch.empty(N // 2, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
def run(with_d2h):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        e[0].record(); d.copy_(h, non_blocking=True); e[1].record()
    if with_d2h:
        with torch.cuda.stream(s2):
            e[2].record(); h2.copy_(d2, non_blocking=True); e[3].record()
    torch.cuda.synchronize()
    t_h2d = e[0].elapsed_time(e[1])
    t_d2h = e[2].elapsed_time(e[3]) if with_d2h else 0
    return t_h2d, t_d2h
for rep in range(3):
    a = run(False); b = run(True)
    print(f"H2D 2 GB alone: {a[0]:.2f} ms ({2*N/a[0]/1e6:.1f} GB/s); with a concurrent 0.5 GB D2H: H2D {b[0]:.2f} ms ({2*N/b[0]/1e6:.1f} GB/s), D2H {b[1]:.2f} ms ({N/2/b[1]/1e6:.1f} GB/s)")
