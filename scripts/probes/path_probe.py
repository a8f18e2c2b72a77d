"""One pairwise step through each kernel path (tn_contract_pair with a forced path),
complex64 or complex128, operands in matricised order; run under
`ncu --metrics gpu__time_duration.sum` for device times (tn_contract_pair builds a plan per
call: its wall time is host work).  python scripts/probes/path_probe.py nb m n k [c64|c128] [path]"""
import sys
import torch
sys.path.insert(0, '.')
import paper_2208_01498_b200 as tb
nb, m, n, k = (int(v) for v in sys.argv[1:5])
c128 = len(sys.argv) > 5 and sys.argv[5] == "c128"
dt, tdt, esz = (tb.TN_C128, torch.complex128, 16) if c128 else (tb.TN_C64, torch.complex64, 8)
dev = torch.device('cuda:0')
ids = list(range(nb + m + n + k))
bt, mm, nn, kk = ids[:nb], ids[nb:nb + m], ids[nb + m:nb + m + n], ids[nb + m + n:]
A = torch.randn(1 << (nb + m + k), dtype=tdt, device=dev)
B = torch.randn(1 << (nb + n + k), dtype=tdt, device=dev)
C = torch.empty(1 << (nb + m + n), dtype=tdt, device=dev)
nbytes = esz * ((1 << (nb + m + k)) + (1 << (nb + n + k)) + (1 << (nb + m + n)))
ref = None
paths = (("auto", tb.TN_PATH_AUTO), ("small", tb.TN_PATH_SMALL), ("skinny", tb.TN_PATH_SKINNY),
         ("wide", tb.TN_PATH_WIDE), ("tc", tb.TN_PATH_TC))
if len(sys.argv) > 6:
    paths = [p for p in paths if p[0] == sys.argv[6]]
for name, path in paths:
    try:
        call = lambda: tb.contract_pair(dt, A.data_ptr(), bt + mm + kk, B.data_ptr(), bt + kk + nn, C.data_ptr(),
                                        bt + mm + nn, [2] * len(ids), path)
        call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if ref is None:
            ref = C.clone()
        err = float((C - ref).abs().max() / ref.abs().max())
        print(f"({nb},{m},{n},{k}) {'c128' if c128 else 'c64'} {name:6s} {ms * 1e3:8.1f} us  {nbytes / ms / 1e9:7.1f} GB/s  rel diff {err:.1e}")
    except Exception as e:
        print(f"({nb},{m},{n},{k}) {name:6s} refused: {str(e)[:80]}")
