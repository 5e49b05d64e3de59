"""One device-resident tprod at config-5 slice shape with a few frequencies (for ncu launch lists)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2212_14318_b200 as qt
m = n = s = int(os.environ.get("OZP_N", 2048)); p = int(os.environ.get("OZP_P", 4))
dev = torch.device("cuda")
mk = lambda r, c: torch.randn(p, r, c, dtype=torch.complex128, device=dev)
a1, a2, b1, b2 = mk(m, n), mk(m, n), mk(n, s), mk(n, s)
c1, c2 = torch.empty(p, m, s, dtype=torch.complex128, device=dev), torch.empty(p, m, s, dtype=torch.complex128, device=dev)
for _ in range(2):
    qt.tprod_fast_device(a1, a2, b1, b2, c1, c2, m, n, s, p)
torch.cuda.synchronize()
print("ok")
