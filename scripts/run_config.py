"""Time full amplitudes of a config on one GPU: python scripts/run_config.py <cfg> [n_bits] [max_log2_size]"""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2208_01498_b200 as tb
from tn_inputs import config_circuit, random_bitstrings, CONFIGS
ci = int(sys.argv[1]); nbits = int(sys.argv[2]) if len(sys.argv) > 2 else 4
tgt = int(sys.argv[3]) if len(sys.argv) > 3 else 0
c = config_circuit(ci)
hyper = ci == 3
dtype = tb.TN_C128 if CONFIGS[ci]["dtype"] == "c128" else tb.TN_C64
t0 = time.time(); net = tb.Network.from_circuit(c, diag_hyper=hyper); order = tb.Order(net, seed=0, max_log2_size=tgt)
t1 = time.time(); plan = tb.Plan(net, order, dtype=dtype); t2 = time.time()
info = plan.info(); oi = order.info()
print(f"config {ci}: order {t1-t0:.2f}s plan {t2-t1:.2f}s  {oi}  {info}")
bits = random_bitstrings(c.n, nbits, 1)
plan.amplitudes(bits[:1])
torch.cuda.synchronize()
t = time.time(); amps = plan.amplitudes(bits); dt = time.time() - t
fl = info['flops_per_slice'] * info['n_slices'] * nbits
print(f"{nbits} amplitudes in {dt:.3f}s: {nbits/dt:.2f} amp/s, {fl/dt/1e12:.2f} TFLOP/s; first {amps[0]}")
