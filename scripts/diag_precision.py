"""Diagnostic: tensor-core complex64 GEMM error relative to |C| and its bias."""
import math, sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2208_01498_b200 as tb
dev = torch.device('cuda:0')
for k in [4, 6, 8, 10, 12]:
    m = n = 7
    ids = list(range(m + n + k)); mm, nn, kk = ids[:m], ids[m:m+n], ids[m+n:]
    g = np.random.default_rng(k)
    A = ((g.standard_normal((1 << m, 1 << k)) + 1j * g.standard_normal((1 << m, 1 << k))) / 2 ** 0.5).astype(np.complex64)
    B = ((g.standard_normal((1 << k, 1 << n)) + 1j * g.standard_normal((1 << k, 1 << n))) / 2 ** 0.5).astype(np.complex64)
    ref = A.astype(np.complex128) @ B.astype(np.complex128)
    for path in (tb.TN_PATH_TC, tb.TN_PATH_SMALL):
        tA, tB = torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev)
        tC = torch.empty((1 << m, 1 << n), dtype=torch.complex64, device=dev)
        tb.contract_pair(tb.TN_C64, tA.data_ptr(), mm + kk, tB.data_ptr(), kk + nn, tC.data_ptr(), mm + nn, [2] * len(ids), path)
        torch.cuda.synchronize()
        got = tC.cpu().numpy().astype(np.complex128)
        rel = np.abs(got - ref) / np.abs(ref)
        bias = np.mean((np.abs(got) - np.abs(ref)) / np.abs(ref))
        print(f"K=2^{k:2d} {'TC   ' if path == tb.TN_PATH_TC else 'small'} rel-to-|C| median {np.median(rel):.2e} "
              f"p99 {np.quantile(rel, .99):.2e}  bias {bias:+.2e}  (2^-24*K/16*12 = {2**-24*12*(1<<k)/16:.1e})")
