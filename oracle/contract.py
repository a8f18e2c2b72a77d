"""Naive contraction along an order (TEST INFRASTRUCTURE -- oracle).

Pairwise contraction of two tensors (Fig. 1b, l.54: "a line connecting two
tensors to a contraction (i.e., a summation) of the corresponding index") along the
step list produced by oracle.ssa.find_order, in complex128.  An index shared by the
two operands is summed iff no tensor outside them still holds it (hyperedges stay as
batch indices); results are stored with indices in ascending id order.

Eq. (3) (l.82-86): a pairwise step costs M multiplications (M = product of the
dimensions of all indices of both operands, shared ones once) and <= M additions.
`contract_pair_loops` executes a step literally and counts both, which pins
oracle.ssa.step_costs.
"""
from __future__ import annotations

import itertools

import numpy as np


def kept_per_step(net, steps):
    """For every step: sorted list of indices kept in its result."""
    n = len(net.tensors)
    total = {}
    nodes = {}
    for t in range(n):
        ii = net.closed_inds(t)
        nodes[t] = {i: 1 for i in ii}
        for i in ii:
            total[i] = total.get(i, 0) + 1
    out = []
    for k, (a, b) in enumerate(steps):
        A, B = nodes.pop(a), nodes.pop(b)
        cnt = dict(A)
        for i, c in B.items():
            cnt[i] = cnt.get(i, 0) + c
        kept = {i: c for i, c in cnt.items() if c < total[i]}
        nodes[n + k] = kept
        out.append(sorted(kept))
    return out


def leaf_tensors(net, bits, fixed=None):
    """Leaf tensors with output legs fixed to the bitstring (and sliced indices fixed
    to the given values): a list of (inds, data)."""
    fix = dict(fixed or {})
    for q in range(net.n_qubits):
        fix[net.out_leg[q]] = int(bits[q])
    out = []
    for T in net.tensors:
        data = T.data
        inds = list(T.inds)
        for ax in range(len(inds) - 1, -1, -1):
            if inds[ax] in fix:
                data = np.take(data, fix[inds[ax]], axis=ax)
                inds.pop(ax)
        out.append((inds, np.asarray(data)))
    return out


def contract_pair(Ainds, A, Binds, B, kept, dims):
    """C[kept sorted] = sum over the other indices of A * B (batch-aware)."""
    kept = set(kept)
    # sum out indices private to one operand that are not kept
    Ai, Bi = list(Ainds), list(Binds)
    for ax in range(len(Ai) - 1, -1, -1):
        if Ai[ax] not in Bi and Ai[ax] not in kept:
            A = A.sum(axis=ax)
            Ai.pop(ax)
    for ax in range(len(Bi) - 1, -1, -1):
        if Bi[ax] not in Ai and Bi[ax] not in kept:
            B = B.sum(axis=ax)
            Bi.pop(ax)
    batch = [i for i in Ai if i in Bi and i in kept]
    contr = [i for i in Ai if i in Bi and i not in kept]
    left = [i for i in Ai if i not in Bi]
    right = [i for i in Bi if i not in Ai]
    d = lambda ii: int(np.prod([dims[i] for i in ii])) if ii else 1
    A2 = np.transpose(A, [Ai.index(i) for i in batch + left + contr]).reshape(d(batch), d(left), d(contr))
    B2 = np.transpose(B, [Bi.index(i) for i in batch + contr + right]).reshape(d(batch), d(contr), d(right))
    C = np.matmul(A2, B2)
    cin = batch + left + right
    C = C.reshape([dims[i] for i in cin]) if cin else C.reshape(())
    out = sorted(cin)
    if out:
        C = np.transpose(C, [cin.index(i) for i in out])
    return out, np.array(C, order="C", copy=True)


def contract_slice(net, steps, bits, fixed, kept=None, keep_intermediates=False):
    """One sliced sub-contraction ("index slicing"): the closed network
    with the output legs bound to `bits` and every sliced index i fixed to fixed[i],
    contracted along `steps`; returns the scalar (and the intermediates if asked)."""
    kept = kept if kept is not None else kept_per_step(net, steps)
    n = len(net.tensors)
    nodes = dict(enumerate(leaf_tensors(net, bits, fixed)))
    inter = [] if keep_intermediates else None
    for k, (a, b) in enumerate(steps):
        (Ai, A), (Bi, B) = nodes.pop(a), nodes.pop(b)
        kk = [i for i in kept[k] if i not in fixed]
        nodes[n + k] = contract_pair(Ai, A, Bi, B, kk, net.dims)
        if keep_intermediates:
            inter.append(nodes[n + k])
    val = 1.0 + 0j
    for inds, data in nodes.values():     # a single root, or disconnected pieces
        assert not inds
        val *= complex(data)
    return (val, inter) if keep_intermediates else val


def contract_tree(net, steps, bits, sliced=(), keep_intermediates=False):
    """<x|C|0> by contracting the closed network along `steps`; sliced indices are
    summed outside the tree (every assignment contracted separately and added)."""
    kept = kept_per_step(net, steps)
    sliced = list(sliced)
    total = 0j
    inter = None
    for vals in itertools.product(*[range(net.dims[i]) for i in sliced]):
        r = contract_slice(net, steps, bits, dict(zip(sliced, vals)), kept, keep_intermediates)
        if keep_intermediates:
            r, inter = r
        total += r
    return (total, inter) if keep_intermediates else total


def contract_pair_loops(Ainds, A, Binds, B, kept, dims):
    """Literal nested-loop execution of one step; returns (result dict, n_mul, n_add).
    n_mul must equal M of Eq. (3); n_add <= M."""
    union = list(dict.fromkeys(list(Ainds) + list(Binds)))
    kept = [i for i in union if i in set(kept)]
    res = {}
    n_mul = 0
    n_add = 0
    for vals in itertools.product(*[range(dims[i]) for i in union]):
        v = dict(zip(union, vals))
        a = A[tuple(v[i] for i in Ainds)]
        b = B[tuple(v[i] for i in Binds)]
        key = tuple(v[i] for i in kept)
        p = a * b
        n_mul += 1
        if key in res:
            res[key] = res[key] + p
            n_add += 1
        else:
            res[key] = p
    return kept, res, n_mul, n_add
