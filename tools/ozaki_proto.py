"""Prototype of the Ozaki-II (CRT) int8 formulation of stage 2, in torch on the GPU.

Research tool only (not the product): validates the integer/CRT math of the paired-frequency
product and measures the library int8 GEMM rate on B200 before the hand-written tcgen05 kernel.
"""
import math
import sys
import time

import numpy as np
import torch

MODULI = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193]


def smod(x, p):  # symmetric residue in [-(p//2), (p-1)//2] (p=256: [-128,127])
    r = torch.remainder(x, p)
    return torch.where(r > (p - 1) // 2, r - p, r)


def crt_signed(res, mods):
    """Garner mixed-radix with signed digits, evaluated top-down in float64."""
    n = len(mods)
    v = []
    for i in range(n):
        p = mods[i]
        t = res[i].to(torch.int64)
        # subtract the value of earlier digits mod p
        acc = torch.zeros_like(t)
        for j in range(i - 1, -1, -1):
            acc = torch.remainder(acc * mods[j] + v[j], p)
        inv = pow(math.prod(mods[:i]) % p, -1, p) if i else 1
        d = torch.remainder((t - acc) * inv, p)
        d = torch.where(d > (p - 1) // 2, d - p, d)
        v.append(d)
    x = torch.zeros_like(v[0], dtype=torch.float64)
    for i in range(n - 1, -1, -1):
        x = x * mods[i] + v[i].to(torch.float64)
    return x


def int_rows(x, b, dim):
    """x (real float64) -> integers round(x * 2^e) with per-row (dim=1) / per-col (dim=0) e."""
    mx = x.abs().amax(dim=dim, keepdim=True)
    _, E = torch.frexp(torch.where(mx > 0, mx, torch.ones_like(mx)))
    e = (b - E).to(torch.int64)
    return torch.round(torch.ldexp(x, e.to(x.dtype))).to(torch.int64), e


def ozaki_pair_product(A1, A2, B1, B2, b=53, nmod=16):
    """A1,A2: (p,m,n) complex128 cuda; B1,B2: (p,n,s). Returns C1,C2 (p,m,s)."""
    p, m, n = A1.shape
    s = B1.shape[2]
    mods = MODULI[:nmod]
    C1 = torch.empty((p, m, s), dtype=torch.complex128, device=A1.device)
    C2 = torch.empty_like(C1)
    for k in range(p):
        sg = (p - k) % p
        X = torch.cat([torch.cat([A1[k], -A2[sg].conj()], 1), torch.cat([A2[k], A1[sg].conj()], 1)], 0)
        Y = torch.cat([B1[k], B2[k]], 0)
        # common exponent over re & im per row of X / column of Y
        XX = torch.cat([X.real, X.imag], 1)
        _, ex = int_rows(XX, b, 1)
        Xr = torch.round(torch.ldexp(X.real, ex.double())).to(torch.int64)
        Xi = torch.round(torch.ldexp(X.imag, ex.double())).to(torch.int64)
        YY = torch.cat([Y.real, Y.imag], 0)
        _, ey = int_rows(YY, b, 0)
        Yr = torch.round(torch.ldexp(Y.real, ey.double())).to(torch.int64)
        Yi = torch.round(torch.ldexp(Y.imag, ey.double())).to(torch.int64)
        Ab = torch.cat([Xr, Xi], 1)                      # 2m x 4n
        Bb = torch.cat([torch.cat([Yr, Yi], 1), torch.cat([-Yi, Yr], 1)], 0)  # 4n x 2s
        res = []
        for q in mods:
            aq = smod(Ab, q).to(torch.int8).contiguous()
            bq = smod(Bb, q).to(torch.int8).t().contiguous().t()
            g = torch._int_mm(aq, bq) if aq.is_cuda else (aq.long() @ bq.long())
            res.append(torch.remainder(g.to(torch.int64), q))
        T = crt_signed(res, mods)
        sc = torch.ldexp(torch.ones_like(T[:, :s]), (-ex - ey).double())
        Re, Im = T[:, :s] * sc, T[:, s:] * sc
        Cc = torch.complex(Re, Im)
        C1[k], C2[k] = Cc[:m], Cc[m:]
    return C1, C2


def bench_int_mm(M, K, N, reps=20):
    a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
    bt = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
    b = bt.t()
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        torch._int_mm(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return ms, 2 * M * K * N / ms / 1e9


def main():
    for (M, K, N) in [(4096, 8192, 4096), (8192, 8192, 8192), (2160, 7680, 128), (512, 1024, 512)]:
        ms, tops = bench_int_mm(M, K, N)
        print(f"int_mm {M}x{K}x{N}: {ms:.3f} ms  {tops:.0f} TOPS", flush=True)
    sys.path.insert(0, ".")
    import paper_2212_14318_b200 as qt
    import oracle as O
    for (m, n, s, p) in [(24, 16, 20, 6), (64, 96, 80, 8), (256, 256, 256, 16)]:
        a = qt.gen_random_tensor(m, n, p, 11)
        bb = qt.gen_random_tensor(n, s, p, 12)
        ah, bh = qt.qfft3_conj(a), qt.qfft3_conj(bb)
        t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
        for nmod, b in [(16, 53), (15, 50), (14, 47)]:
            C1, C2 = ozaki_pair_product(t(ah.t1), t(ah.t2), t(bh.t1), t(bh.t2), b=b, nmod=nmod)
            c = qt.qifft3_conj(qt.CdTensor3(m, s, p, C1.cpu().numpy(), C2.cpu().numpy()))
            ref = O.tprod_fast((a.t1, a.t2), (bb.t1, bb.t2))
            gpu = qt.tprod_fast(a, bb)
            e_oz = O.rel_frob_error((c.t1, c.t2), ref)
            e_dm = O.rel_frob_error((gpu.t1, gpu.t2), ref)
            if m * n * s * p <= 24 * 16 * 20 * 6 * 20:
                nv = O.tprod_naive((a.t1, a.t2), (bb.t1, bb.t2))
                extra = f" | vs naive: ozaki {O.rel_frob_error((c.t1, c.t2), nv):.2e} dmma {O.rel_frob_error((gpu.t1, gpu.t2), nv):.2e} ref {O.rel_frob_error(ref, nv):.2e}"
            else:
                extra = ""
            print(f"({m},{n},{s},{p}) nmod={nmod} b={b}: ozaki vs ref {e_oz:.2e}; dmma vs ref {e_dm:.2e}{extra}", flush=True)


if __name__ == "__main__":
    main()
