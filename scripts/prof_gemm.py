"""One tensor-core contraction step (pack x2 + cgemm) at a config-1-like shape, for ncu.
usage: python scripts/prof_gemm.py m n k [nb]   (TN_PROF_PATH=wide|skinny|small|tc, default tc)"""
import sys
import torch
sys.path.insert(0, '.')
import paper_2208_01498_b200 as tb
m, n, k = (int(v) for v in sys.argv[1:4])
nb = int(sys.argv[4]) if len(sys.argv) > 4 else 0
dev = torch.device('cuda:0')
import os
path = {'tc': tb.TN_PATH_TC, 'wide': tb.TN_PATH_WIDE, 'skinny': tb.TN_PATH_SKINNY, 'small': tb.TN_PATH_SMALL}[os.environ.get('TN_PROF_PATH', 'tc')]
ids = list(range(nb + m + n + k))
bt, mm, nn, kk = ids[:nb], ids[nb:nb + m], ids[nb + m:nb + m + n], ids[nb + m + n:]
A = torch.randn(1 << (nb + m + k), dtype=torch.complex64, device=dev)
B = torch.randn(1 << (nb + n + k), dtype=torch.complex64, device=dev)
C = torch.empty(1 << (nb + m + n), dtype=torch.complex64, device=dev)
for _ in range(2):
    tb.contract_pair(tb.TN_C64, A.data_ptr(), bt + mm + kk, B.data_ptr(), bt + kk + nn, C.data_ptr(), bt + mm + nn,
                     [2] * len(ids), path)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
tb.contract_pair(tb.TN_C64, A.data_ptr(), bt + mm + kk, B.data_ptr(), bt + kk + nn, C.data_ptr(), bt + mm + nn,
                 [2] * len(ids), path)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"step m={m} n={n} k={k} nb={nb}: {ms:.3f} ms (pack+gemm), {8 * 2.0 ** (nb + m + n + k) / ms / 1e9:.1f} TFLOP/s")
