"""Timing probe: the configs[1] dominant pair-GEMM step (16, 16, 12) run back to back
(power-capped steady state), device time per launch by CUDA events.  Used with the normal
library and with one where mma_loop_pair skipped its fourth MMA per split term (an
`#ifndef TN_PROBE_MMA9` around the `t_im += a_im b_re` issue, built with
TN_NVCC_EXTRA=-DTN_PROBE_MMA9; wrong results, removed after the measurement): 9 of the
12 MMAs per K step, the tensor work of a 3-real-product (Gauss) complex scheme, to see
how the step time scales with the MMA count."""
import sys, time
import torch
sys.path.insert(0, '.')
import paper_2208_01498_b200 as tb
m, n, k = 16, 16, 12
dev = torch.device('cuda:0')
ids = list(range(m + n + k))
mm, nn, kk = ids[:m], ids[m:m + n], ids[m + n:]
A = torch.randn(1 << (m + k), dtype=torch.complex64, device=dev)
B = torch.randn(1 << (n + k), dtype=torch.complex64, device=dev)
C = torch.empty(1 << (m + n), dtype=torch.complex64, device=dev)
ts = []
for r in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tb.contract_pair(tb.TN_C64, A.data_ptr(), mm + kk, B.data_ptr(), kk + nn, C.data_ptr(), mm + nn, [2] * len(ids),
                     tb.TN_PATH_TC)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("ms per step (pack + GEMM):", " ".join(f"{t:.1f}" for t in ts))
