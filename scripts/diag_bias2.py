"""Relative bias of the complex64 tensor-core GEMM (RZ accumulation in TMEM) per K and
operand distribution: bias = Re(sum conj(ref)(got - ref)) / sum |ref|^2, in units of
2^-24.  python scripts/diag_bias2.py"""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2208_01498_b200 as tb
dev = torch.device('cuda:0')


def gen(g, shape, kind):
    z = (g.standard_normal(shape) + 1j * g.standard_normal(shape)) / 2 ** 0.5
    if kind == "lognormal":
        z = z * np.exp(1.5 * g.standard_normal(shape))
    elif kind == "sparse":
        z = z * (g.random(shape) < 0.3)
    elif kind == "phase":       # unit-modulus entries
        z = np.exp(2j * np.pi * g.random(shape))
    return z.astype(np.complex64)


for kind in ("gauss", "lognormal", "sparse", "phase"):
    for (m, n, k) in ((9, 8, 4), (9, 8, 5), (9, 8, 6), (9, 8, 7), (9, 8, 10), (7, 7, 6), (7, 7, 10), (10, 10, 12)):
        ids = list(range(m + n + k)); mm, nn, kk = ids[:m], ids[m:m + n], ids[m + n:]
        g = np.random.default_rng(100 * k + m)
        A, B = gen(g, (1 << m, 1 << k), kind), gen(g, (1 << k, 1 << n), kind)
        tA, tB = torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev)
        ref = tA.to(torch.complex128) @ tB.to(torch.complex128)
        tC = torch.empty((1 << m, 1 << n), dtype=torch.complex64, device=dev)
        tb.contract_pair(tb.TN_C64, tA.data_ptr(), mm + kk, tB.data_ptr(), kk + nn, tC.data_ptr(), mm + nn, [2] * len(ids),
                         tb.TN_PATH_TC)
        torch.cuda.synchronize()
        err = tC.to(torch.complex128) - ref
        den = (ref.abs() ** 2).sum()
        bias = float((ref.conj() * err).real.sum() / den) / 2 ** -24
        rms = float((err.abs() ** 2).sum().sqrt() / den.sqrt()) / 2 ** -24
        print(f"{kind:9s} m={m:2d} n={n:2d} K=2^{k:2d}: bias {bias:+7.2f}  rms {rms:6.2f}  (x 2^-24)", flush=True)
