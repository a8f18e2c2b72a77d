"""Skinny steps of a config's plan, each run through tn_contract_pair (v2 kernel) under a watchdog.
python scripts/skinny_shapes.py <config> [target]"""
import sys, subprocess, os
sys.path.insert(0, '.')
import paper_2208_01498_b200 as tb
from tn_inputs import config_circuit, CONFIGS
ci = int(sys.argv[1]); tgt = int(sys.argv[2]) if len(sys.argv) > 2 else 0
c = config_circuit(ci)
net = tb.Network.from_circuit(c, diag_hyper=(ci == 3))
o = tb.Order(net, seed=0, max_log2_size=tgt)
dt = tb.TN_C64 if CONFIGS[ci]["dtype"] == "c64" else tb.TN_C128
p = tb.Plan(net, o, dtype=dt)
shapes = sorted({tuple(int(v) for v in r[1:5]) for r in p.steps() if int(r[0]) == tb.TN_PATH_SKINNY})
print("skinny shapes (nb, m, n, k):", shapes, flush=True)
for nb, m, n, k in shapes:
    code = f"""
import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import test_gpu as T, paper_2208_01498_b200 as tb, numpy as np
ia, ib, ic, dims = T._gemm_case({nb}, {m}, {n}, {k})
got, ref, bound = T._run_pair(ia, ib, ic, dims, {dt}, tb.TN_PATH_SKINNY)
print('max err/bound', float((abs(got - ref) / (bound + 1e-300)).max()))
"""
    try:
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=60)
        print((nb, m, n, k), r.stdout.strip()[-80:], r.stderr.strip()[-200:], flush=True)
    except subprocess.TimeoutExpired:
        print((nb, m, n, k), "TIMEOUT (hang)", flush=True)
