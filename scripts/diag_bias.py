"""Relative bias and rms error of the complex64 tensor-core GEMM vs complex128, per K:
bias = Re(sum conj(ref) (got - ref)) / sum |ref|^2  (a uniform shrink shows as < 0).
python scripts/diag_bias.py [m] [n] [ks...]"""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2208_01498_b200 as tb
dev = torch.device('cuda:0')
m = int(sys.argv[1]) if len(sys.argv) > 1 else 9
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
ks = [int(v) for v in sys.argv[3:]] or [5, 7, 9, 11, 13, 15]
for k in ks:
    ids = list(range(m + n + k)); mm, nn, kk = ids[:m], ids[m:m + n], ids[m + n:]
    g = np.random.default_rng(k)
    A = ((g.standard_normal((1 << m, 1 << k)) + 1j * g.standard_normal((1 << m, 1 << k))) / 2 ** 0.5).astype(np.complex64)
    B = ((g.standard_normal((1 << k, 1 << n)) + 1j * g.standard_normal((1 << k, 1 << n))) / 2 ** 0.5).astype(np.complex64)
    tA, tB = torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev)
    ref = (tA.to(torch.complex128) @ tB.to(torch.complex128))
    for path in (tb.TN_PATH_TC,):
        tC = torch.empty((1 << m, 1 << n), dtype=torch.complex64, device=dev)
        tb.contract_pair(tb.TN_C64, tA.data_ptr(), mm + kk, tB.data_ptr(), kk + nn, tC.data_ptr(), mm + nn, [2] * len(ids), path)
        torch.cuda.synchronize()
        err = tC.to(torch.complex128) - ref
        bias = float((ref.conj() * err).real.sum() / (ref.abs() ** 2).sum())
        rms = float((err.abs() ** 2).sum().sqrt() / (ref.abs() ** 2).sum().sqrt())
        T = 48 if k >= 7 else 12 * (1 << (k - 5))
        print(f"m={m} n={n} K=2^{k:2d}: bias {bias:+.3e} = {bias / 2**-24:+7.2f} x 2^-24   rms {rms:.3e} = {rms / 2**-24:6.2f} x 2^-24", flush=True)
