import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2212_14318_b200 as qt
from paper_2212_14318_b200 import _native
m, n, s, p = [int(v) for v in os.environ.get("OZD", "4,64,4,5").split(",")]
rng = np.random.default_rng(0)
cx = lambda *sh: rng.standard_normal(sh) + 1j * rng.standard_normal(sh)
A1, A2, B1, B2 = cx(p, m, n), cx(p, m, n), cx(p, n, s), cx(p, n, s)
t = lambda x: torch.from_numpy(x).cuda()
a1, a2, b1, b2 = t(A1), t(A2), t(B1), t(B2)
c1 = torch.zeros(p, m, s, dtype=torch.complex128, device="cuda"); c2 = torch.zeros_like(c1)
L = _native.lib()
rc = L.qt_spectral_product_f64_device(a1.data_ptr(), a2.data_ptr(), b1.data_ptr(), b2.data_ptr(), c1.data_ptr(), c2.data_ptr(), m, n, s, p, None)
print("rc", rc)
torch.cuda.synchronize()
C1, C2 = c1.cpu().numpy(), c2.cpu().numpy()
for k in range(p):
    sk = (p - k) % p
    R1 = A1[k] @ B1[k] - np.conj(A2[sk]) @ B2[k]
    R2 = np.conj(A1[sk]) @ B2[k] + A2[k] @ B1[k]
    e1 = np.linalg.norm(C1[k] - R1) / np.linalg.norm(R1); e2 = np.linalg.norm(C2[k] - R2) / np.linalg.norm(R2)
    print(k, f"{e1:.2e} {e2:.2e}")
