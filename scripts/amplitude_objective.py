"""Would an order objective that counts slice reuse and provably zero slices pick another
hierarchy than R10 (least sliced work)?  Over all n_seeds hierarchies of the oracle:
amplitude work = invariant + contributing slices x per-slice dependent work, for the bench
batch's first bitstring.  python scripts/amplitude_objective.py <config> <target> <n_seeds>"""
import sys, math, itertools, multiprocessing as mp
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import numpy as np
from tn_inputs import config_circuit, random_bitstrings
from oracle.network import build_network
from oracle import ssa

ci = int(sys.argv[1]); tgt = int(sys.argv[2]); nseeds = int(sys.argv[3])
net = build_network(config_circuit(ci))
n = len(net.tensors)
l2 = {i: net.log2dim(i) for i in range(len(net.dims))}
outs = {leg: q for q, leg in enumerate(net.out_leg)}
x = random_bitstrings(net.n_qubits, 1024, 1)[0]

def analyze(r):
    tot, steps, log = ssa._one_hierarchy((net, 0, 8, 32, 64, 256, tgt, r))
    sl = ssa.choose_slices(net, steps, tgt)
    sls = set(sl)
    # invariant vs dependent Eq.(3) work per slice
    dep = {t: any(i in sls for i in net.tensors[t].inds) for t in range(n)}
    nodes = {}; total = {}
    for t in range(n):
        nodes[t] = {i: 1 for i in net.closed_inds(t)}
        for i in nodes[t]: total[i] = total.get(i, 0) + 1
    inv_w = dep_w = 0.0
    for k, (a, b) in enumerate(steps):
        A, B = nodes[a], nodes[b]; cnt = dict(A)
        for i, c in B.items(): cnt[i] = cnt.get(i, 0) + c
        m = sum(l2[i] for i in cnt if i not in sls)
        nodes[n + k] = {i: c for i, c in cnt.items() if c < total[i]}
        dep[n + k] = dep[a] or dep[b]
        if dep[n + k]: dep_w += 2.0 ** m
        else: inv_w += 2.0 ** m
    # provably zero slices for bitstring x: a leaf whose only sliced index is j
    allowed = {i: set(range(net.dims[i])) for i in sl}
    for t, T in enumerate(net.tensors):
        sidx = [i for i in T.inds if i in sls]
        if len(sidx) != 1: continue
        j = sidx[0]
        d = T.data
        # fix output legs to x
        idx = []
        for ax, i in enumerate(T.inds):
            idx.append(int(x[outs[i]]) if i in outs else slice(None))
        sub = d[tuple(idx)]
        rem = [i for i in T.inds if i not in outs]
        axj = rem.index(j)
        sub = np.moveaxis(sub, axj, 0).reshape(net.dims[j], -1)
        nz = {v for v in range(net.dims[j]) if np.any(sub[v] != 0)}
        allowed[j] &= nz
    contrib = 1.0
    for i in sl: contrib *= len(allowed[i])
    sb = sum(l2[i] for i in sl)
    amp = inv_w + contrib * dep_w
    return r, math.log2(tot), sb, contrib, math.log2(amp), math.log2((inv_w + dep_w) * contrib)

with mp.Pool(8) as p:
    res = p.map(analyze, range(nseeds), chunksize=1)
res.sort(key=lambda t: t[1])
best_r10 = res[0]
best_amp = min(res, key=lambda t: t[4])
print("R10 choice (min sliced work):", best_r10)
print("min amplitude work with reuse + zero slices:", best_amp)
print("ratio", 2 ** (best_r10[4] - best_amp[4]))
