"""Independent pins of the separator steps of oracle/ssa.py (CPU, -m "not gpu").

Every check recomputes what the paper fixes from the raw network (positions, radius,
index lists) with plain loops written here, never from ssa.py's own counts:
  * SST statement: every separator S splits the spheres into
    Gamma_O (spheres S meets), Gamma_E, Gamma_I with Eq. (1) |Gamma_O| <= c_2 k^{1/2} n^{1/2}
    and Eq. (2) |Gamma_E|, |Gamma_I| <= 3n/4, and Gamma_E, Gamma_I mutually non-intersecting;
  * SM Algorithm 1 step 7 (l.206): the check "taking account of the radii";
  * Theorem 1 proof (l.79): each Gamma_O tensor joins the side with which it shares
    indices of higher overall bond dimension (ties: arbitrary -- our R7 tie rule), so it
    shares at most half its index bits, <= log2 M^{1/2}, with the other side;
  * Theorem 2 proof (l.122-123): connected tensors have intersecting spheres; the
    overlap bound k = F((l/4 + r/4)/(r/4))^2 for the single-copy network (R8);
  * SM "Numerical implementation" (l.217): the greedy leaf planner merges, at every
    step, a pair of minimum Eq. (3) cost M among the pairs sharing an index (R9).
"""
import math
import random

import numpy as np
import pytest

from tn_inputs import lattice_cz, sycamore, random3d, iqp
from oracle.network import build_network
from oracle import ssa
from oracle.rng import Stream


# ----------------------------------------------------------- helpers (plain) --
def _log2(d):
    b = 0
    while (1 << b) < d:
        b += 1
    assert (1 << b) == d
    return b


def _closed(net, t):
    outs = set(net.out_leg)
    return [i for i in net.tensors[t].inds if i not in outs]


def _label(sep, x, y, r):
    """Where the ball of radius r at (x, y) lies relative to the separator S:
    'O' if S meets it, else the side.  Circle (cx, cy, rho): interior 'I' iff the
    farthest point of the ball is inside, exterior 'E' iff the nearest point is outside.
    Line {p : 2 b.p = C0}: the side of the ball's centre if the centre is farther than r."""
    if sep[0] == "circle":
        _, cx, cy, rho = sep
        d = math.hypot(x - cx, y - cy)
        if d + r < rho:
            return "I"
        if d - r > rho:
            return "E"
        return "O"
    _, b0, b1, c0, _nb = sep
    nb = math.hypot(b0, b1)
    # foot of the perpendicular from the origin: p0 = (c0 / 2) b / |b|^2
    p0x, p0y = 0.5 * c0 * b0 / (nb * nb), 0.5 * c0 * b1 / (nb * nb)
    signed = ((x - p0x) * b0 + (y - p0y) * b1) / nb
    if signed > r:
        return "+"
    if signed < -r:
        return "-"
    return "O"


def _hierarchy(net, seed=0, root=1):
    ctx = ssa._Ctx(net, seed, 8, 32, 64, 256)
    ssa._build(ctx, list(range(len(net.tensors))), root, 0)
    return ctx


NETS = {
    "lattice6x6d8": lambda: build_network(lattice_cz(6, 6, 8, 3)),
    "lattice5x7d12": lambda: build_network(lattice_cz(5, 7, 12, 4)),
    "sycamore_m4": lambda: build_network(sycamore(4, 5)),
    "random3d_8": lambda: build_network(random3d(8, 6, 6, n_patches=1, patch=4)),
}


def _net(name, cache={}):
    if name not in cache:
        cache[name] = NETS[name]()
    return cache[name]


# --------------------------------------------------- Theorem 2 construction --
@pytest.mark.parametrize("name", sorted(NETS))
def test_connected_tensors_have_intersecting_spheres(name):
    """Theorem 1 hypothesis as built in the Theorem 2 proof: spheres of tensors with a
    contracted index intersect (centre distance <= 2 radius)."""
    net = _net(name)
    r = net.radius
    holders = {}
    for t in range(len(net.tensors)):
        for i in _closed(net, t):
            holders.setdefault(i, []).append(t)
    n_pairs = 0
    for i, ts in holders.items():
        for a in range(len(ts)):
            for b in range(a + 1, len(ts)):
                pa, pb = net.tensors[ts[a]].pos, net.tensors[ts[b]].pos
                assert math.hypot(pa[0] - pb[0], pa[1] - pb[1]) <= 2 * r, (i, ts[a], ts[b])
                n_pairs += 1
    assert n_pairs > 0


def test_k_bound_and_radius_closed_form_on_lattice():
    """Nearest-neighbour lattice of spacing 1 (l = r = 1): radius l/4 + eps, and
    k = F (1 + l/r)^2 = 4F with F = max number of two-qubit gates on one qubit."""
    c = lattice_cz(4, 5, 9, 2)
    net = build_network(c)
    per_q = [0] * c.n
    for qs, _ in c.gates:
        if len(qs) == 2:
            per_q[qs[0]] += 1
            per_q[qs[1]] += 1
    assert net.k_bound == 4.0 * max(per_q)
    assert abs(net.radius - (0.25 + 0.01)) < 1e-15


# ----------------------------------------------------------- classification --
def test_classify_closed_form_cases():
    """Hand-placed balls against the unit circle and the line x = 1/2."""
    circ = ("circle", 0.0, 0.0, 1.0)
    PX = np.array([0.0, 0.75, 0.95, 1.05, 1.25, 3.0, 0.0])
    PY = np.array([0.0, 0.0, 0.0, 0.0, 0.0, 0.0, -0.85])
    want = [2, 2, 0, 0, 1, 1, 0]          # 2 = I, 1 = E, 0 = O
    assert list(ssa.classify(circ, PX, PY, 0.2)) == want
    # radius halved: the balls at 0.95 and 1.05 are still cut, the one at distance 0.85 is inside
    assert list(ssa.classify(circ, PX, PY, 0.1)) == [2, 2, 0, 0, 1, 1, 2]
    # line 2 (b . p) = C0 with b = (1, 0), C0 = 1  ->  x = 1/2
    line = ("line", 1.0, 0.0, 1.0, 1.0)
    PX = np.array([0.0, 0.4, 0.6, 1.0])
    labs = list(ssa.classify(line, PX, np.zeros(4), 0.2))
    assert labs[1] == 0 and labs[2] == 0
    assert labs[0] != 0 and labs[3] != 0 and labs[0] != labs[3]


@pytest.mark.parametrize("name", sorted(NETS))
def test_every_separator_satisfies_sst(name):
    """Every SSA split of a whole hierarchy, re-classified here: Eqs. (1)-(2), the
    step-7 radius check, Gamma_E / Gamma_I non-intersecting, and E / I as returned
    are Gamma_E / Gamma_I plus the Gamma_O tensors."""
    net = _net(name)
    ctx = _hierarchy(net)
    r = net.radius
    k = net.k_bound
    assert ctx.seps, "no SSA separator in the hierarchy"
    for ids, sep, E, I in ctx.seps:
        s = len(ids)
        lab = {t: _label(sep, net.tensors[t].pos[0], net.tensors[t].pos[1], r) for t in ids}
        sides = sorted({v for v in lab.values() if v != "O"})
        O = [t for t in ids if lab[t] == "O"]
        if sep[0] == "circle":
            inner = [t for t in ids if lab[t] == "I"]
            outer = [t for t in ids if lab[t] == "E"]
        else:
            inner = [t for t in ids if lab[t] == "-"]
            outer = [t for t in ids if lab[t] == "+"]
            if not (set(outer) <= set(E)):
                inner, outer = outer, inner
        assert set(outer) <= set(E) and set(inner) <= set(I), (sep, sides)
        assert sorted(E + I) == sorted(ids) and not set(E) & set(I)
        assert set(E) - set(outer) | set(I) - set(inner) == set(O)
        # Eq. (1), d = 2, c_2 = 2
        assert len(O) <= 2.0 * math.sqrt(k) * math.sqrt(s), (len(O), k, s)
        # Eq. (2), (d+1)/(d+2) = 3/4
        assert 4 * len(outer) <= 3 * s and 4 * len(inner) <= 3 * s, (len(outer), len(inner), s)
        # Gamma_E and Gamma_I do not intersect
        for a in outer:
            pa = net.tensors[a].pos
            for b in inner:
                pb = net.tensors[b].pos
                assert math.hypot(pa[0] - pb[0], pa[1] - pb[1]) > 2 * r


@pytest.mark.parametrize("name", sorted(NETS))
def test_boundary_assignment_follows_theorem1(name):
    """Theorem 1 proof (l.79) on every split: replaying the decisions over the returned
    sides, each Gamma_O tensor (ascending id, R7) went to the side with which it shares
    more index bits (ties: the smaller side, then E), so at its decision it shares at
    most half of its own index bits -- <= log2 M^{1/2} -- with the other side."""
    net = _net(name)
    ctx = _hierarchy(net)
    r = net.radius
    n_O = n_tie = 0
    for ids, sep, E, I in ctx.seps:
        lab = {t: _label(sep, net.tensors[t].pos[0], net.tensors[t].pos[1], r) for t in ids}
        Eset = set(E) - {t for t in ids if lab[t] == "O"}
        Iset = set(I) - {t for t in ids if lab[t] == "O"}
        for t in sorted(t for t in ids if lab[t] == "O"):
            inds = _closed(net, t)
            held_E = {i for u in Eset for i in _closed(net, u)}
            held_I = {i for u in Iset for i in _closed(net, u)}
            wE = sum(_log2(net.dims[i]) for i in inds if i in held_E)
            wI = sum(_log2(net.dims[i]) for i in inds if i in held_I)
            to_E = t in E
            if wE != wI:
                assert to_E == (wE > wI), (t, wE, wI)
            else:
                n_tie += 1
                assert to_E == (len(Eset) <= len(Iset)), (t, len(Eset), len(Iset))
            bits = sum(_log2(net.dims[i]) for i in inds)
            assert 2 * (wI if to_E else wE) <= bits
            (Eset if to_E else Iset).add(t)
            n_O += 1
    assert n_O > 0


def test_separator_on_10x10_grid_satisfies_eqs_1_2():
    """10x10 lattice network, one SSA call on all tensors: the returned separator,
    re-classified here, meets Eqs. (1)-(2) and the counts ssa reports are those."""
    c = lattice_cz(10, 10, 4, 71)
    net = build_network(c)
    ctx = ssa._Ctx(net, 0, 8, 32, 8, 64)
    ids = list(range(len(net.tensors)))
    res = ssa.find_separator(ctx, ids, Stream(0, 1))
    assert res is not None
    E, I, key, tries, (nO, nE, nI), sep = res
    s = len(ids)
    lab = [_label(sep, net.tensors[t].pos[0], net.tensors[t].pos[1], net.radius) for t in ids]
    cnt = {v: lab.count(v) for v in set(lab)}
    assert cnt.get("O", 0) == nO
    assert nO <= 2.0 * math.sqrt(net.k_bound) * math.sqrt(s)
    assert 4 * nE <= 3 * s and 4 * nI <= 3 * s
    assert sorted(E + I) == ids and E and I


# -------------------------------------------------------------- greedy leaves --
def _replay_greedy(net, ids, steps, n0):
    """Check every merge of greedy_leaf against all candidate pairs (R9): the chosen
    pair shares an index if any pair does and minimises (log2 M, log2 result, ids)."""
    total = {}
    for t in range(len(net.tensors)):
        for i in _closed(net, t):
            total[i] = total.get(i, 0) + 1
    cur = {t: {i: 1 for i in _closed(net, t)} for t in ids}
    for k, (a, b) in enumerate(steps):
        keys = {}
        any_shared = False
        for x in cur:
            for y in cur:
                if x >= y:
                    continue
                shared = bool(set(cur[x]) & set(cur[y]))
                union = set(cur[x]) | set(cur[y])
                M = sum(_log2(net.dims[i]) for i in union)
                res = sum(_log2(net.dims[i]) for i in union if cur[x].get(i, 0) + cur[y].get(i, 0) < total[i])
                keys[(x, y)] = (shared, M, res, x, y)
                any_shared = any_shared or shared
        cands = [v[1:] for v in keys.values() if v[0] or not any_shared]
        chosen = keys[(min(a, b), max(a, b))]
        assert chosen[0] or not any_shared, "merged a pair without a shared index"
        assert chosen[1:] == min(cands), (k, chosen, min(cands))
        A, B = cur.pop(a), cur.pop(b)
        m = dict(A)
        for i, c in B.items():
            m[i] = m.get(i, 0) + c
        cur[n0 + k] = {i: c for i, c in m.items() if c < total[i]}


@pytest.mark.parametrize("name", sorted(NETS))
def test_greedy_leaf_merges_minimum_cost_pair(name):
    net = _net(name)
    n = len(net.tensors)
    hier = _hierarchy(net)
    leaves = list(hier.leaves[:12])
    # plus random connected clusters of 4..8 tensors
    rnd = random.Random(7)
    nbr = {t: set() for t in range(n)}
    holders = {}
    for t in range(n):
        for i in _closed(net, t):
            holders.setdefault(i, []).append(t)
    for ts in holders.values():
        for a in ts:
            nbr[a].update(u for u in ts if u != a)
    for _ in range(8):
        start = rnd.randrange(n)
        cl = [start]
        while len(cl) < rnd.randint(4, 8):
            fr = sorted({u for t in cl for u in nbr[t]} - set(cl))
            if not fr:
                break
            cl.append(rnd.choice(fr))
        leaves.append(sorted(cl))
    for ids in leaves:
        ctx = ssa._Ctx(net, 0, 8, 32, 64, 256)
        ssa.greedy_leaf(ctx, list(ids))
        assert len(ctx.steps) == len(ids) - 1
        _replay_greedy(net, ids, ctx.steps, n)


def _check_split(net, ids, res, k):
    E, I, key, tries, (nO, nE, nI), sep = res
    s = len(ids)
    lab = [_label(sep, net.tensors[t].pos[0], net.tensors[t].pos[1], net.radius) for t in ids]
    O = lab.count("O")
    sides = [lab.count(v) for v in sorted(set(lab) - {"O"})]
    assert (O, sorted(sides + [0] * (2 - len(sides)))) == (nO, sorted([nE, nI]))
    assert O * O <= 4.0 * k * s, (O, k, s)                  # Eq. (1), c_2 = 2
    assert all(4 * v <= 3 * s for v in sides), (sides, s)    # Eq. (2)


def test_step7_accepts_only_circles_satisfying_eqs_1_2():
    """Algorithm 1 step 7 on its own: with n_valid = 1 the FIRST accepted great circle is
    returned, so every returned split must pass the check.  Many streams and node sets
    (the whole network and random halves of it).  Half of the trials use centerpoints of
    4-point subsets (a_max = 4): poor centerpoints, so ~10% of the circles split 3:4 .. 7:8
    and only the check keeps them out."""
    net = build_network(lattice_cz(8, 8, 6, 9))
    n = len(net.tensors)
    rnd = random.Random(3)
    n_res = 0
    for trial in range(40):
        ctx = ssa._Ctx(net, trial, 8, 4 if trial % 4 < 2 else 32, 1, 256)
        if trial % 2:
            x0 = rnd.uniform(1.0, 6.0)
            ids = [t for t in range(n) if net.tensors[t].pos[0] <= x0] or list(range(n))
        else:
            ids = list(range(n))
        res = ssa.find_separator(ctx, ids, Stream(trial, 5))
        if res is None:
            continue
        _check_split(net, ids, res, net.k_bound)
        n_res += 1
    assert n_res >= 30


def test_step7_eq1_binds_with_small_k():
    """Eq. (1) is loose for circuit networks (k = 4F); shrinking k in the check makes it
    bind: only circles cutting at most 2 k^{1/2} s^{1/2} spheres may be returned."""
    net = build_network(lattice_cz(8, 8, 6, 9))
    n_res = 0
    for trial in range(12):
        ctx = ssa._Ctx(net, trial, 8, 32, 1, 256)
        net.k_bound, k_old = 0.2, net.k_bound
        try:
            res = ssa.find_separator(ctx, list(range(len(net.tensors))), Stream(trial, 6))
        finally:
            net.k_bound = k_old
        if res is None:
            continue
        _check_split(net, list(range(len(net.tensors))), res, 0.2)
        n_res += 1
    assert n_res >= 8


def test_step7_selection_keeps_the_best_valid_circle():
    """R6: among the valid circles the one with the smallest (open bits of the larger
    child, cut) is kept.  The circle sequence of a stream does not depend on n_valid, so
    the key kept with n_valid = 64 is <= the key of the first valid circle (n_valid = 1),
    and both are the (max open bits, cut) of the returned sides, recounted here."""
    net = build_network(lattice_cz(7, 7, 8, 12))
    ids = list(range(len(net.tensors)))
    total = {}
    for t in ids:
        for i in _closed(net, t):
            total[i] = total.get(i, 0) + 1
    n_less = 0
    for trial in range(10):
        r1 = ssa.find_separator(ssa._Ctx(net, 0, 8, 32, 1, 256), ids, Stream(trial, 8))
        r64 = ssa.find_separator(ssa._Ctx(net, 0, 8, 32, 64, 256), ids, Stream(trial, 8))
        for r in (r1, r64):
            E, I = r[0], r[1]
            hE = {i for t in E for i in _closed(net, t)}
            hI = {i for t in I for i in _closed(net, t)}
            cut = sum(_log2(net.dims[i]) for i in hE & hI)
            openE = sum(_log2(net.dims[i]) for i in hE if sum(1 for t in E if i in _closed(net, t)) < total[i])
            openI = sum(_log2(net.dims[i]) for i in hI if sum(1 for t in I if i in _closed(net, t)) < total[i])
            assert r[2] == (max(openE, openI), cut)
        assert r64[2] <= r1[2]
        n_less += r64[2] < r1[2]
    assert n_less >= 3


def test_median_split_fallback():
    """R6 fallback: halves by the coordinate of the wider axis (ties by id)."""
    net = build_network(lattice_cz(3, 6, 4, 2))      # 6 columns: x is the wider axis
    ctx = ssa._Ctx(net, 0, 8, 32, 64, 256)
    ids = list(range(len(net.tensors)))
    E, I = ssa.median_split(ctx, ids)
    assert len(E) == len(ids) // 2 and sorted(E + I) == ids
    assert max(net.tensors[t].pos[0] for t in E) <= min(net.tensors[t].pos[0] for t in I)
