"""Separator-based contraction order (TEST INFRASTRUCTURE -- oracle).

Sphere Separator Algorithm, SM Algorithm 1, for d = 2:
  step 1  stereographic projection Pi: R^2 -> S^2, Pi(q) = (2q, |q|^2-1)/(|q|^2+1)
  step 2  centerpoint c of a random subset S (|S| = a) by linear programming on the
          O(a^{d+1}) half-space inequalities induced by planes through d+1 points of S
  step 3  orthogonal R with R c = (0, 0, |c|)   (Householder reflection)
  step 4  dilatation D_alpha = Pi o (alpha 1) o Pi^{-1}, alpha = sqrt((1-|c|)/(1+|c|))
  step 5  random great circle C (uniform normal u on S^2)
  step 6  S = Pi^{-1} o R^T o D_alpha^{-1}(C)  (a circle or line in R^2, closed form)
  step 7  check Eqs. (1)-(2) taking the radii into account,
          else draw another great circle.
Theorem 1 proof (l.79-80): the spheres cut by S (Gamma_O) are assigned to the side
with which they share indices of higher overall bond dimension; recurse until the
pieces have O(1) tensors (leaf_size).  Leaves are ordered greedily (SM l.217).

All arithmetic that decides the order is written as explicit, left-to-right
IEEE-754 double operations (no BLAS, no pairwise sums, no FMA) so that the C++
implementation, written independently to the same recipe, produces the identical
order.  Readings:
  R5  subset size a = min(s, 32); the LP maximises the margin t of the centerpoint
      inside every heavy half-space (|open side| < a/(d+2)) within the box |c_i| <= 2;
      dual revised simplex, Bland's rule.
  R6  among the first n_valid (64) circles satisfying Eqs. (1)-(2) with two non-empty
      sides, keep the one whose larger child has the fewest open index bits, then the
      smallest cut sum(log2 dim) between the sides (ties: earliest); up to 256 circles
      per centerpoint, 2 centerpoints; if none is valid, median split along the wider
      axis.
  R7  boundary assignment in ascending tensor id against the current sides (already
      assigned boundary tensors count); ties -> smaller side, then E.
  R8  k in Eq. (1) is the Theorem 2 bound F((l+r)/r)^2 (amplitude network: U only).
  R9  greedy leaf planner: among pairs sharing an index (else all pairs) minimise
      log2 of the Eq. (3) cost M, then log2 result size, then (id_i, id_j).
  R10 the randomized hierarchy is built n_seeds (4) times; the one with the smallest
      Eq. (3) total is kept -- of all slices when a slicing target is set.
"""
from __future__ import annotations

import math

import numpy as np

from .rng import Stream, child_stream

BOX = 2.0
LP_TOL = 1e-9
PIV_TOL = 1e-12
SIDE_TOL = 1e-12
C_D = {1: 1.0, 2: 2.0, 3: 2.135, 4: 2.280, 5: 2.421}


# ---------------------------------------------------------------- geometry ---
def stereo(px, py):
    """Step 1, Pi(q) = (2q, |q|^2 - 1)/(|q|^2 + 1) (vectorised, elementwise)."""
    s = px * px + py * py
    den = s + 1.0
    return (2.0 * px) / den, (2.0 * py) / den, (s - 1.0) / den


def inv4(B):
    """Gauss-Jordan inverse of a 4x4 (list of lists) with partial pivoting."""
    M = [list(B[r]) + [1.0 if c == r else 0.0 for c in range(4)] for r in range(4)]
    for col in range(4):
        piv = col
        best = abs(M[col][col])
        for r in range(col + 1, 4):
            if abs(M[r][col]) > best:
                best = abs(M[r][col])
                piv = r
        if best == 0.0:
            return None
        M[col], M[piv] = M[piv], M[col]
        p = M[col][col]
        M[col] = [v / p for v in M[col]]
        for r in range(4):
            if r == col:
                continue
            f = M[r][col]
            if f != 0.0:
                M[r] = [M[r][k] - f * M[col][k] for k in range(8)]
    return [row[4:] for row in M]


def lp_centerpoint(A0, A1, A2, A3, b, maxit=500):
    """max t s.t. A x <= b, x = (c0, c1, c2, t) free; solved on the dual
    min b.y s.t. A^T y = e_t, y >= 0 by revised simplex with Bland's rule.
    Rows 0-2: c_i <= BOX, rows 3-5: -c_i <= BOX, row 6: t <= 1."""
    m = len(b)
    basis = [0, 1, 2, 6]
    pi = None
    for _ in range(maxit):
        B = [[0.0] * 4 for _ in range(4)]
        for c, j in enumerate(basis):
            B[0][c], B[1][c], B[2][c], B[3][c] = A0[j], A1[j], A2[j], A3[j]
        Binv = inv4(B)
        if Binv is None:
            break
        cB = [b[j] for j in basis]
        pi = []
        for i in range(4):
            acc = cB[0] * Binv[0][i]
            for r in range(1, 4):
                acc = acc + cB[r] * Binv[r][i]
            pi.append(acc)
        d = b - (((pi[0] * A0 + pi[1] * A1) + pi[2] * A2) + pi[3] * A3)
        d[basis] = 0.0
        cand = np.nonzero(d < -LP_TOL)[0]
        if cand.size == 0:
            break
        e = int(cand[0])
        Ae = (A0[e], A1[e], A2[e], A3[e])
        best_r, best_theta = -1, 0.0
        for r in range(4):
            w = Binv[r][0] * Ae[0]
            for i in range(1, 4):
                w = w + Binv[r][i] * Ae[i]
            if w > PIV_TOL:
                th = Binv[r][3] / w
                if best_r < 0 or th < best_theta or (th == best_theta and basis[r] < basis[best_r]):
                    best_r, best_theta = r, th
        if best_r < 0:
            break
        basis[best_r] = e
    return pi


def centerpoint(P0, P1, P2, rng: Stream, a_max=32):
    """Step 2: centerpoint of a random subset of the projected points."""
    s = len(P0)
    a = min(s, a_max)
    perm = list(range(s))
    for i in range(a):
        j = i + rng.below(s - i)
        perm[i], perm[j] = perm[j], perm[i]
    S = perm[:a]
    X = np.array([P0[i] for i in S])
    Y = np.array([P1[i] for i in S])
    Z = np.array([P2[i] for i in S])
    rows0 = [1.0, 0.0, 0.0, -1.0, 0.0, 0.0, 0.0]
    rows1 = [0.0, 1.0, 0.0, 0.0, -1.0, 0.0, 0.0]
    rows2 = [0.0, 0.0, 1.0, 0.0, 0.0, -1.0, 0.0]
    rows3 = [0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 1.0]
    rb = [BOX] * 6 + [1.0]
    if a >= 3:
        ii, jj, kk = [], [], []
        for i in range(a):
            for j in range(i + 1, a):
                for k in range(j + 1, a):
                    ii.append(i)
                    jj.append(j)
                    kk.append(k)
        ii, jj, kk = np.array(ii), np.array(jj), np.array(kk)
        ux, uy, uz = X[jj] - X[ii], Y[jj] - Y[ii], Z[jj] - Z[ii]
        vx, vy, vz = X[kk] - X[ii], Y[kk] - Y[ii], Z[kk] - Z[ii]
        nx = uy * vz - uz * vy
        ny = uz * vx - ux * vz
        nz = ux * vy - uy * vx
        nn2 = (nx * nx + ny * ny) + nz * nz
        ok = nn2 > 1e-24
        nrm = np.sqrt(np.where(ok, nn2, 1.0))
        nx, ny, nz = nx / nrm, ny / nrm, nz / nrm
        off = (nx * X[ii] + ny * Y[ii]) + nz * Z[ii]
        side = ((nx[:, None] * X[None, :] + ny[:, None] * Y[None, :]) + nz[:, None] * Z[None, :]) - off[:, None]
        above = (side > SIDE_TOL).sum(axis=1)
        below = (side < -SIDE_TOL).sum(axis=1)
        for t in range(len(ii)):
            if not ok[t]:
                continue
            if above[t] * 4 < a:
                rows0.append(float(nx[t])); rows1.append(float(ny[t])); rows2.append(float(nz[t]))
                rows3.append(1.0); rb.append(float(off[t]))
            if below[t] * 4 < a:
                rows0.append(float(-nx[t])); rows1.append(float(-ny[t])); rows2.append(float(-nz[t]))
                rows3.append(1.0); rb.append(float(-off[t]))
    pi = lp_centerpoint(np.array(rows0), np.array(rows1), np.array(rows2), np.array(rows3), np.array(rb))
    if pi is None:
        return (0.0, 0.0, 0.0)
    c = (pi[0], pi[1], pi[2])
    nc = math.sqrt((c[0] * c[0] + c[1] * c[1]) + c[2] * c[2])
    if nc > 0.999999:
        f = 0.999999 / nc
        c = (c[0] * f, c[1] * f, c[2] * f)
    return c


def rotation_to_pole(c):
    """Step 3: Householder R with R c = (0, 0, |c|)."""
    I = [[1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]]
    nc = math.sqrt((c[0] * c[0] + c[1] * c[1]) + c[2] * c[2])
    if nc < 1e-12:
        return I, 0.0
    v = (c[0] / nc, c[1] / nc, c[2] / nc)
    w = (v[0], v[1], v[2] - 1.0)
    ww = (w[0] * w[0] + w[1] * w[1]) + w[2] * w[2]
    if ww < 1e-24:
        return I, nc
    R = [[I[r][k] - (2.0 * w[r] * w[k]) / ww for k in range(3)] for r in range(3)]
    return R, nc


def random_normal(rng: Stream):
    """Step 5: uniform direction on S^2 by rejection from the cube."""
    while True:
        u0 = 2.0 * rng.uniform() - 1.0
        u1 = 2.0 * rng.uniform() - 1.0
        u2 = 2.0 * rng.uniform() - 1.0
        r2 = (u0 * u0 + u1 * u1) + u2 * u2
        if 1e-6 < r2 <= 1.0:
            r = math.sqrt(r2)
            return (u0 / r, u1 / r, u2 / r)


def separator_circle(u, R, alpha):
    """Step 6 in closed form.  C = {z : u.z = 0}.  D_alpha^{-1}(C) lies on the plane
    n.z = h with n = (alpha u0, alpha u1, u2 (1+alpha^2)/2), h = u2 (1-alpha^2)/2;
    R^T maps it to the plane (R^T n).z = h; Pi^{-1} of the plane (n, h) is
    A|p|^2 + 2 b.p - C0 = 0 with A = n2 - h, b = (n0, n1), C0 = n2 + h."""
    a2 = alpha * alpha
    n = (alpha * u[0], alpha * u[1], (u[2] * (1.0 + a2)) / 2.0)
    h = (u[2] * (1.0 - a2)) / 2.0
    m = [(R[0][i] * n[0] + R[1][i] * n[1]) + R[2][i] * n[2] for i in range(3)]
    A = m[2] - h
    b0, b1 = m[0], m[1]
    C0 = m[2] + h
    scale = ((abs(A) + abs(b0)) + abs(b1)) + abs(C0)
    if abs(A) > 1e-12 * scale:
        cx, cy = -b0 / A, -b1 / A
        rho2 = (b0 * b0 + b1 * b1) / (A * A) + C0 / A
        if not rho2 > 0.0:
            return None
        return ("circle", cx, cy, math.sqrt(rho2))
    nb = math.sqrt(b0 * b0 + b1 * b1)
    if nb == 0.0:
        return None
    return ("line", b0, b1, C0, nb)


def classify(sep, PX, PY, rad):
    """Gamma_O / Gamma_E / Gamma_I of the SST (l.45): 0 = O (sphere meets S),
    1 = E (exterior), 2 = I (interior); vectorised over tensors."""
    if sep[0] == "circle":
        _, cx, cy, rho = sep
        dx, dy = PX - cx, PY - cy
        dist = np.sqrt(dx * dx + dy * dy)
        lab = np.zeros(len(PX), dtype=np.int64)
        lab[dist + rad < rho] = 2
        lab[dist - rad > rho] = 1
        return lab
    _, b0, b1, C0, nb = sep
    sd = (2.0 * (b0 * PX + b1 * PY) - C0) / (2.0 * nb)
    lab = np.zeros(len(PX), dtype=np.int64)
    lab[sd > rad] = 1
    lab[sd < -rad] = 2
    return lab


# ------------------------------------------------------------- hierarchy ----
class _Ctx:
    def __init__(self, net, seed, leaf_size, a_max, n_valid, max_tries):
        self.net = net
        self.seed = seed
        self.leaf_size = leaf_size
        self.a_max = a_max
        self.n_valid = n_valid
        self.max_tries = max_tries
        self.inds = [net.closed_inds(t) for t in range(len(net.tensors))]
        self.l2 = {i: net.log2dim(i) for i in range(len(net.dims))}
        self.PX = np.array([T.pos[0] for T in net.tensors], dtype=np.float64)
        self.PY = np.array([T.pos[1] for T in net.tensors], dtype=np.float64)
        self.total = {}
        for t, ii in enumerate(self.inds):
            for i in ii:
                self.total[i] = self.total.get(i, 0) + 1
        self.steps = []
        self.n_leaves = len(net.tensors)
        self.log = []
        self.seps = []        # (ids, separator, E, I) of every SSA split, for the pins
        self.leaves = []      # ids of every greedy leaf, for the pins


def assign_boundary(ctx, ids, lab):
    """Theorem 1 proof (l.79): each Gamma_O tensor joins the side with which it
    shares indices of higher overall bond dimension (R7)."""
    cntE, cntI = {}, {}
    E, I, O = [], [], []
    for t, l in zip(ids, lab):
        (O if l == 0 else E if l == 1 else I).append(t)
    for t in E:
        for i in ctx.inds[t]:
            cntE[i] = cntE.get(i, 0) + 1
    for t in I:
        for i in ctx.inds[t]:
            cntI[i] = cntI.get(i, 0) + 1
    for t in O:
        wE = 0
        wI = 0
        for i in ctx.inds[t]:
            if cntE.get(i, 0) > 0:
                wE += ctx.l2[i]
            if cntI.get(i, 0) > 0:
                wI += ctx.l2[i]
        if wE > wI:
            side = 1
        elif wI > wE:
            side = 2
        else:
            side = 1 if len(E) <= len(I) else 2
        if side == 1:
            E.append(t)
            for i in ctx.inds[t]:
                cntE[i] = cntE.get(i, 0) + 1
        else:
            I.append(t)
            for i in ctx.inds[t]:
                cntI[i] = cntI.get(i, 0) + 1
    cut = 0
    openE = 0
    openI = 0
    for i, c in cntE.items():
        if cntI.get(i, 0) > 0:
            cut += ctx.l2[i]
        if c < ctx.total[i]:
            openE += ctx.l2[i]
    for i, c in cntI.items():
        if c < ctx.total[i]:
            openI += ctx.l2[i]
    return sorted(E), sorted(I), (max(openE, openI), cut)


def find_separator(ctx, ids, rng):
    """Algorithm 1 steps 1-7 on the tensors `ids`; returns None or
    (E, I, (max open bits, cut), tries, (|O|, |E|, |I|), separator)."""
    s = len(ids)
    PX = ctx.PX[ids]
    PY = ctx.PY[ids]
    P0, P1, P2 = stereo(PX, PY)
    rad = ctx.net.radius
    k = ctx.net.k_bound
    best = None
    n_ok = 0
    tries = 0
    for _round in range(2):
        c = centerpoint(list(P0), list(P1), list(P2), rng, ctx.a_max)
        R, nc = rotation_to_pole(c)
        alpha = math.sqrt((1.0 - nc) / (1.0 + nc))
        for _ in range(ctx.max_tries):
            tries += 1
            u = random_normal(rng)
            sep = separator_circle(u, R, alpha)
            if sep is None:
                continue
            lab = classify(sep, PX, PY, rad)
            nO = int((lab == 0).sum())
            nE = int((lab == 1).sum())
            nI = int((lab == 2).sum())
            # Eq. (1): |Gamma_O| <= c_d k^{1/d} n^{1-1/d}  (d = 2: |O|^2 <= 4 k s)
            if not float(nO * nO) <= (C_D[2] * C_D[2]) * k * float(s):
                continue
            # Eq. (2): |Gamma_E|, |Gamma_I| <= (d+1)/(d+2) n  (d = 2: 4|.| <= 3 s)
            if 4 * nE > 3 * s or 4 * nI > 3 * s:
                continue
            E, I, cut = assign_boundary(ctx, ids, lab)
            if not E or not I:
                continue
            n_ok += 1
            if best is None or cut < best[2]:
                best = (E, I, cut, tries, (nO, nE, nI), sep)
            if n_ok >= ctx.n_valid:
                break
        if best is not None:
            break
    return best


def median_split(ctx, ids):
    PX = ctx.PX[ids]
    PY = ctx.PY[ids]
    wx = float(PX.max() - PX.min())
    wy = float(PY.max() - PY.min())
    key = PX if wx >= wy else PY
    order = sorted(range(len(ids)), key=lambda j: (float(key[j]), ids[j]))
    h = len(ids) // 2
    E = sorted(ids[j] for j in order[:h])
    I = sorted(ids[j] for j in order[h:])
    return E, I


class _Node:
    __slots__ = ("nid", "counts")

    def __init__(self, nid, counts):
        self.nid = nid
        self.counts = counts      # index -> number of original holders inside


def _merge(ctx, A: _Node, B: _Node) -> _Node:
    counts = dict(A.counts)
    for i, c in B.counts.items():
        counts[i] = counts.get(i, 0) + c
    kept = {i: c for i, c in counts.items() if c < ctx.total[i]}
    nid = ctx.n_leaves + len(ctx.steps)
    ctx.steps.append((A.nid, B.nid))
    return _Node(nid, kept)


def greedy_leaf(ctx, ids):
    """SM 'Numerical implementation' (l.217): greedy pairwise order of a leaf (R9)."""
    cur = [_Node(t, {i: 1 for i in ctx.inds[t]}) for t in ids]
    while len(cur) > 1:
        best = None
        share_any = False
        cands = []
        for x in range(len(cur)):
            for y in range(x + 1, len(cur)):
                A, B = cur[x], cur[y]
                shared = any(i in B.counts for i in A.counts)
                cands.append((shared, x, y))
                share_any = share_any or shared
        for shared, x, y in cands:
            if share_any and not shared:
                continue
            A, B = cur[x], cur[y]
            union = set(A.counts) | set(B.counts)
            cost = sum(ctx.l2[i] for i in union)
            res = 0
            for i in union:
                if A.counts.get(i, 0) + B.counts.get(i, 0) < ctx.total[i]:
                    res += ctx.l2[i]
            key = (cost, res, min(A.nid, B.nid), max(A.nid, B.nid))
            if best is None or key < best[0]:
                best = (key, x, y)
        _, x, y = best
        A, B = cur[x], cur[y]
        if A.nid > B.nid:
            A, B = B, A
        node = _merge(ctx, A, B)
        cur = [c for j, c in enumerate(cur) if j != x and j != y] + [node]
    return cur[0]


def _build(ctx, ids, sid, depth):
    if len(ids) <= ctx.leaf_size:
        ctx.leaves.append(list(ids))
        return greedy_leaf(ctx, ids)
    rng = Stream(ctx.seed, sid)
    res = find_separator(ctx, ids, rng)
    if res is None:
        E, I = median_split(ctx, ids)
        ctx.log.append((depth, len(ids), "median"))
    else:
        E, I, cut, tries, _cnt, sep = res
        ctx.log.append((depth, len(ids), cut, tries))
        ctx.seps.append((list(ids), sep, E, I))
    nE = _build(ctx, E, child_stream(sid, 0), depth + 1)
    nI = _build(ctx, I, child_stream(sid, 1), depth + 1)
    return _merge(ctx, nE, nI)


def _one_hierarchy(args):
    """One randomized hierarchy (root stream 1 + r) and its R10 objective."""
    net, seed, leaf_size, a_max, n_valid, max_tries, max_log2_size, r = args
    ctx = _Ctx(net, seed, leaf_size, a_max, n_valid, max_tries)
    ids = list(range(len(net.tensors)))
    _build(ctx, ids, 1 + r, 0)
    tot = 0.0
    for m, _ in step_costs(net, ctx.steps):
        tot = tot + 2.0 ** (m + 1)
    if max_log2_size > 0:
        tot = sliced_work(net, ctx.steps, choose_slices(net, ctx.steps, max_log2_size))
    return tot, ctx.steps, ctx.log


def find_order(net, seed: int = 0, leaf_size: int = 8, a_max: int = 32, n_valid: int = 64,
               max_tries: int = 256, n_seeds: int = 4, max_log2_size: int = 0, map_fn=map):
    """Separator hierarchy (Fig. 2) -> list of pairwise steps (a, b); leaves are
    tensor ids 0..n-1, step k creates node id n + k.  Post-order: E subtree, I
    subtree, then their merge.  The randomized hierarchy is built n_seeds times
    (root stream ids 1..n_seeds) and the one with the smallest Eq. (3) total
    sum_k 2 M_k is kept -- with a slicing target, the smallest total of all slices,
    sliced_work(choose_slices(...)) (R10; ties -> earliest).  The hierarchies are
    independent; `map_fn` (e.g. a process pool's map, order-preserving) builds them."""
    best = None
    args = [(net, seed, leaf_size, a_max, n_valid, max_tries, max_log2_size, r) for r in range(n_seeds)]
    for tot, steps, log in map_fn(_one_hierarchy, args):
        if best is None or tot < best[0]:
            best = (tot, steps, log)
    return best[1], best[2]


def sliced_work(net, steps, slices):
    """Eq. (3) work of all slices, W = 2^{sum sliced bits} * sum_k 2^{m_k - sliced bits
    of step k} (left to right, doubles): what the greedy slicer (R11) minimises."""
    n = len(net.tensors)
    l2 = {i: net.log2dim(i) for i in range(len(net.dims))}
    sl = set(slices)
    total = {}
    nodes = {}
    for t in range(n):
        ii = net.closed_inds(t)
        nodes[t] = {i: 1 for i in ii}
        for i in ii:
            total[i] = total.get(i, 0) + 1
    w = 0.0
    for k, (a, b) in enumerate(steps):
        A, B = nodes.pop(a), nodes.pop(b)
        cnt = dict(A)
        for i, c in B.items():
            cnt[i] = cnt.get(i, 0) + c
        nodes[n + k] = {i: c for i, c in cnt.items() if c < total[i]}
        m = sum(l2[i] for i in sorted(cnt))
        s = sum(l2[i] for i in sorted(cnt) if i in sl)
        w = w + 2.0 ** (m - s)
    return w * 2.0 ** sum(l2[i] for i in sl)


def step_costs(net, steps):
    """log2 of M^{(l+1)} of Eq. (3) for every step (product of the dimensions of all
    indices of the two operands, shared ones counted once) and log2 result size."""
    n = len(net.tensors)
    l2 = {i: net.log2dim(i) for i in range(len(net.dims))}
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
        union = set(A) | set(B)
        cnt = {i: A.get(i, 0) + B.get(i, 0) for i in union}
        kept = {i: c for i, c in cnt.items() if c < total[i]}
        nodes[n + k] = kept
        out.append((sum(l2[i] for i in union), sum(l2[i] for i in kept)))
    return out


def choose_slices(net, steps, max_log2_size: int):
    """Index slicing (the outlook's "index slicing approach"; BASELINE
    north_star "index slicing splits one contraction into independent sliced
    sub-contractions").  Greedy (R11): while some tensor of the contraction (leaf or
    intermediate) has more than max_log2_size index bits after removing the sliced
    indices, slice the index -- among those held by such a largest tensor -- that
    minimises the total Eq. (3) work of all slices
        W = 2^{sum sliced bits} * sum_k 2^{m_k - sliced bits of step k}
    (summed left to right over steps, doubles), ties -> smaller index id.
    Returns the sorted list of sliced indices."""
    n = len(net.tensors)
    l2 = {i: net.log2dim(i) for i in range(len(net.dims))}
    total = {}
    nodes = {}
    tensors = []          # index sets of every tensor that ever exists
    for t in range(n):
        ii = net.closed_inds(t)
        nodes[t] = {i: 1 for i in ii}
        tensors.append(sorted(ii))
        for i in ii:
            total[i] = total.get(i, 0) + 1
    step_union = []
    for k, (a, b) in enumerate(steps):
        A, B = nodes.pop(a), nodes.pop(b)
        cnt = dict(A)
        for i, c in B.items():
            cnt[i] = cnt.get(i, 0) + c
        kept = {i: c for i, c in cnt.items() if c < total[i]}
        nodes[n + k] = kept
        step_union.append(sorted(cnt))
        tensors.append(sorted(kept))
    step_m = [sum(l2[i] for i in u) for u in step_union]
    sliced = set()

    def bits(ii):
        return sum(l2[i] for i in ii if i not in sliced)

    while True:
        big = max(bits(ii) for ii in tensors)
        if big <= max_log2_size:
            break
        cands = sorted({i for ii in tensors if bits(ii) == big for i in ii if i not in sliced})
        best = None
        sb = sum(l2[i] for i in sliced)
        for c in cands:
            w = 0.0
            for u, m in zip(step_union, step_m):
                s = 0
                for i in u:
                    if i in sliced or i == c:
                        s += l2[i]
                w = w + 2.0 ** (m - s)
            w = w * 2.0 ** (sb + l2[c])
            if best is None or w < best[0]:
                best = (w, c)
        sliced.add(best[1])
    return sorted(sliced)
