"""Step paths of a config's plan: python scripts/plan_summary.py <config> <slice target> [n_seeds]"""
import sys
import collections
sys.path.insert(0, '.')
import paper_2208_01498_b200 as tb
from tn_inputs import config_circuit, CONFIGS
ci, tgt = int(sys.argv[1]), int(sys.argv[2])
ns = int(sys.argv[3]) if len(sys.argv) > 3 else 256
c = config_circuit(ci)
net = tb.Network.from_circuit(c, diag_hyper=(ci == 3))
o = tb.Order(net, seed=0, n_seeds=ns, max_log2_size=tgt)
p = tb.Plan(net, o, dtype=tb.TN_C64 if CONFIGS[ci]["dtype"] == "c64" else tb.TN_C128)
st = p.steps()
names = {0: "auto", 1: "small", 2: "tc", 3: "skinny", 4: "wide"}
cnt = collections.Counter(int(r[0]) for r in st)
fl = collections.Counter()
for r in st:
    fl[int(r[0])] += 8.0 * 2.0 ** int(r[1] + r[2] + r[3] + r[4])
tot = sum(fl.values())
print(f"config {ci} target {tgt}: {p.info()}")
for k in sorted(cnt):
    print(f"  {names.get(k, k)}: {cnt[k]} steps, {fl[k] / tot:.4f} of flops")
big = sorted(st, key=lambda r: -int(r[1] + r[2] + r[3] + r[4]))[:25]
for r in big:
    print("   ", names.get(int(r[0])), "nb,m,n,k =", tuple(int(v) for v in r[1:5]), "share %.4f" % (8.0 * 2.0 ** int(r[1] + r[2] + r[3] + r[4]) / tot))
