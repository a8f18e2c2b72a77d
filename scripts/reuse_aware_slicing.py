"""Would a reuse-aware greedy slicer (objective: prologue work once + slice-dependent work per
slice, R16) choose better sliced indices than R11 (all work per slice)?  Oracle only:
python scripts/reuse_aware_slicing.py <config> (uses oracle/orders/config<ci>.json)."""
import json, sys, math
sys.path.insert(0, '.')
from tn_inputs import config_circuit
from oracle.network import build_network
ci = int(sys.argv[1])
d = json.load(open(f'oracle/orders/config{ci}.json'))
net = build_network(config_circuit(ci), diag_hyper=d['diag_hyper'])
steps = [tuple(s) for s in d['steps']]
n = len(net.tensors)
l2 = {i: net.log2dim(i) for i in range(len(net.dims))}
total = {}; nodes = {}; tensors = []; leaves_of = {}
for t in range(n):
    ii = net.closed_inds(t); nodes[t] = {i: 1 for i in ii}; tensors.append(sorted(ii)); leaves_of[t] = set(ii)
    for i in ii: total[i] = total.get(i, 0) + 1
step_union = []; sub_inds = []   # all indices held by leaves of the subtree
for k, (a, b) in enumerate(steps):
    A, B = nodes.pop(a), nodes.pop(b)
    cnt = dict(A)
    for i, c in B.items(): cnt[i] = cnt.get(i, 0) + c
    kept = {i: c for i, c in cnt.items() if c < total[i]}
    nodes[n + k] = kept; step_union.append(sorted(cnt)); tensors.append(sorted(kept))
    leaves_of[n + k] = leaves_of[a] | leaves_of[b]; sub_inds.append(leaves_of[n + k])
step_m = [sum(l2[i] for i in u) for u in step_union]
def works(sliced):
    sb = sum(l2[i] for i in sliced)
    pro = dep = 0.0
    for u, m, si in zip(step_union, step_m, sub_inds):
        s = sum(l2[i] for i in u if i in sliced)
        w = 2.0 ** (m - s)
        if si & sliced: dep += w
        else: pro += w
    return pro, dep, sb
def greedy(max_log2, reuse):
    sliced = set()
    bits = lambda ii: sum(l2[i] for i in ii if i not in sliced)
    while True:
        big = max(bits(ii) for ii in tensors)
        if big <= max_log2: break
        cands = sorted({i for ii in tensors if bits(ii) == big for i in ii if i not in sliced})
        best = None
        for c in cands:
            pro, dep, sb = works(sliced | {c})
            w = (pro + dep * 2.0 ** sb) if reuse else (pro + dep) * 2.0 ** sb
            if best is None or w < best[0]: best = (w, c)
        sliced.add(best[1])
    return sliced
for reuse in (False, True):
    s = greedy(d['max_log2_size'], reuse)
    pro, dep, sb = works(s)
    print('reuse-aware' if reuse else 'current    ', 'sliced bits', sb, 'log2 amp work (reuse):', round(math.log2(pro + dep * 2 ** sb), 2), 'pro', round(math.log2(pro),2) if pro else None, 'dep/slice', round(math.log2(dep), 2), 'no reuse', round(math.log2((pro + dep) * 2 ** sb), 2))
print('file slices', d['slices'] if isinstance(d['slices'], int) else len(d['slices']))
