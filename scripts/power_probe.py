"""Board power and SM clock (NVML, 10 ms) during (a) an HBM-bound copy loop and (b) the
tensor-core GEMM of one bench-shaped step: does the memory-bound phase run below the
power cap?  usage: python scripts/power_probe.py"""
import sys, threading, time
sys.path.insert(0, '.')
import numpy as np, torch, pynvml as nv
import paper_2208_01498_b200 as tb

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
limit = nv.nvmlDeviceGetEnforcedPowerLimit(h) / 1000.0


def sample(fn, seconds=4.0):
    rows, stop = [], threading.Event()
    def poll():
        while not stop.is_set():
            rows.append((nv.nvmlDeviceGetPowerUsage(h) / 1000.0, nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
            time.sleep(0.01)
    t = threading.Thread(target=poll); t.start()
    t0 = time.time(); n = 0
    while time.time() - t0 < seconds:
        fn(); n += 1
    torch.cuda.synchronize(); stop.set(); t.join()
    rows = rows[len(rows) // 4:]          # skip the ramp
    return np.median([r[0] for r in rows]), np.median([r[1] for r in rows]), n


dev = torch.device('cuda:0')
x = torch.empty(2 << 30, dtype=torch.float32, device=dev); y = torch.empty_like(x)
p, c, n = sample(lambda: y.copy_(x))
print(f"copy 8 GB loop: power {p:.0f} W (limit {limit:.0f} W), SM clock {c:.0f} MHz")
del x, y; torch.cuda.empty_cache()
m, nn, k = 14, 12, 14
ids = list(range(m + nn + k))
A = torch.randn(1 << (m + k), dtype=torch.complex64, device=dev)
B = torch.randn(1 << (nn + k), dtype=torch.complex64, device=dev)
C = torch.empty(1 << (m + nn), dtype=torch.complex64, device=dev)
f = lambda: tb.contract_pair(tb.TN_C64, A.data_ptr(), ids[:m] + ids[m + nn:], B.data_ptr(), ids[m + nn:] + ids[m:m + nn],
                             C.data_ptr(), ids[:m + nn], [2] * len(ids), tb.TN_PATH_TC)
p, c, n = sample(f)
print(f"tensor-core step (2^{m}, 2^{nn}, 2^{k}) loop: power {p:.0f} W, SM clock {c:.0f} MHz")
