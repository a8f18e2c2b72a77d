import sys, os, time; sys.path.insert(0, '.')
import numpy as np, paper_2208_01498_b200 as tb
from tn_inputs import config_circuit, random_bitstrings
c = config_circuit(1)
net = tb.Network.from_circuit(c)
tgt = int(sys.argv[1]); ns = int(sys.argv[2])
o = tb.Order(net, seed=0, n_seeds=ns, max_log2_size=tgt)
p = tb.Plan(net, o, dtype=tb.TN_C64)
print("slice bits", p.info()["slice_bits"], "arena", p.info()["arena_bytes"] / 1e9)
x = random_bitstrings(c.n, 1, 1)[0]
for s in range(4):
    t = time.time(); a = p.contract(x, s, s + 1); print(s, a, "%.2fs" % (time.time() - t))
x0 = np.zeros(c.n, np.uint8)
print("x=0 slice 0", p.contract(x0, 0, 1))
