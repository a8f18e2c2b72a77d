"""Power-capped steady state of one tensor-core step: the step (pack + GEMM) back to back,
device time per call by CUDA events, useful TF/s.  python scripts/probes/gemm_b2b.py m n k [reps]"""
import sys
import torch
sys.path.insert(0, '.')
import paper_2208_01498_b200 as tb
m, n, k = (int(v) for v in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 8
dev = torch.device('cuda:0')
ids = list(range(m + n + k))
mm, nn, kk = ids[:m], ids[m:m + n], ids[m + n:]
A = torch.randn(1 << (m + k), dtype=torch.complex64, device=dev)
B = torch.randn(1 << (n + k), dtype=torch.complex64, device=dev)
C = torch.empty(1 << (m + n), dtype=torch.complex64, device=dev)
ts = []
for r in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tb.contract_pair(tb.TN_C64, A.data_ptr(), mm + kk, B.data_ptr(), kk + nn, C.data_ptr(), mm + nn, [2] * len(ids),
                     tb.TN_PATH_TC)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
med = sorted(ts[1:])[len(ts[1:]) // 2]
print(f"({m},{n},{k}) median {med:.1f} ms = {8 * 2.0 ** (m + n + k) / med / 1e9:.1f} TF/s useful; all:",
      " ".join(f"{t:.0f}" for t in ts))
