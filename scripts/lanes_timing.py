"""amplitudes/s of configs[3] (and [0]) through tn_amplitudes with 1..8 lanes"""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_2208_01498_b200 as tb
from tn_inputs import config_circuit, random_bitstrings
for ci, dt, hyper in ((3, tb.TN_C128, True), (0, tb.TN_C128, False)):
    c = config_circuit(ci)
    net = tb.Network.from_circuit(c, diag_hyper=hyper)
    plan = tb.Plan(net, tb.Order(net, seed=0), dtype=dt)
    bits = random_bitstrings(c.n, 256, 1)
    ref = None
    for L in (1, 2, 4, 8):
        plan.set_lanes(L)
        plan.amplitudes(bits[:16])
        torch.cuda.synchronize()
        t = time.perf_counter(); a = plan.amplitudes(bits); dt_s = time.perf_counter() - t
        ref = a if ref is None else ref
        print(f"config {ci}: {L} lanes: {len(bits) / dt_s:.1f} amplitudes/s (max |diff| vs 1 lane {abs(a - ref).max():.2e})")
