"""Circuit -> closed tensor network for <x|C|0> (TEST INFRASTRUCTURE -- oracle).

Follows PAPER.md "Classical Simulation of Quantum Circuits" (l.115-125):
  * single-qubit gates are rank-2 tensors, two-qubit gates rank-4 tensors (l.116);
  * single-qubit gates, the |0> inputs (and here the <x| outputs, which stay open
    legs until a bitstring is chosen) are absorbed into the two-qubit gate tensors
    (l.116 "can be absorbed into the former");
  * every two-qubit gate is split into two rank-3 tensors joined by a bond of
    dimension <= 4 (Theorem 2 proof, l.122), placed at x_i + (x_j - x_i)/4 and
    x_j + (x_i - x_j)/4 with sphere radius l/4 + eps (l.122).

Readings:
  R1  split: diagonal gates G = diag(g) use the exact rank-2 split
      X[a',a,s] = d(a'=a=s), Y[b',b,s] = d(b'=b) g(s,b); any other gate the exact
      rank-4 split X[a',a,s] = d(s = 2a'+a), Y[b',b,s] = G[2(s>>1)+b', 2(s&1)+b]
      (same bond dimensions as the SVD of l.122 for the configs' gate families,
      without the SVD's gauge freedom).
  R2  absorption target: a non-core tensor merges into the alive tensor sharing an
      index with it that was created next after it ("chronologically nearest
      later"), else the latest earlier one; passes in creation order repeat until
      none merges.
  R3  optional diagonal simplification (diag_hyper=True, used for IQP): diagonal
      gates keep the wire index unchanged (a hyperedge); a diagonal 2-qubit gate is
      one rank-2 tensor g[z_a, z_b] placed at the Y-half position.
  R4  an index held by a single tensor (and not an output leg) is summed out.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Tensor:
    inds: list            # index ids, in data-axis order
    data: np.ndarray      # complex128, shape = dims of inds
    pos: tuple            # (x, y)
    core: bool
    created: int          # creation slot (used by absorption rule R2)


@dataclass
class Network:
    dims: list                    # index id -> dimension
    tensors: list                 # final tensors (id order), Tensor objects
    out_leg: list                 # qubit q -> index id of its open output leg
    out_owner: list               # qubit q -> tensor id holding that leg
    radius: float                 # sphere radius l/4 + eps
    k_bound: float                # overlap bound used in Eq. (1)
    n_qubits: int
    extras: dict = field(default_factory=dict)

    def closed_inds(self, t: int):
        outs = set(self.out_leg)
        return [i for i in self.tensors[t].inds if i not in outs]

    def log2dim(self, i: int) -> int:
        d = self.dims[i]
        l = d.bit_length() - 1
        assert (1 << l) == d, "dimensions are powers of two"
        return l


def _is_diag(U):
    return bool(np.all(U[~np.eye(U.shape[0], dtype=bool)] == 0))


def _pair_contract(A: Tensor, B: Tensor, keep: set, tie_order):
    """Contract B into A: result axes = A's kept indices (A order) then B's new kept
    indices (B order).  Plain einsum over named indices."""
    letters = {}
    for i in list(A.inds) + list(B.inds):
        if i not in letters:
            letters[i] = chr(ord('a') + len(letters)) if len(letters) < 26 else chr(ord('A') + len(letters) - 26)
    out = [i for i in A.inds if i in keep] + [i for i in B.inds if i in keep and i not in A.inds]
    spec = "".join(letters[i] for i in A.inds) + "," + "".join(letters[i] for i in B.inds) + "->" + \
        "".join(letters[i] for i in out)
    data = np.einsum(spec, A.data, B.data)
    return out, data


def build_network(circ, diag_hyper: bool = False, eps_frac: float = 0.01) -> Network:
    n = circ.n
    pos = np.asarray(circ.pos, dtype=np.float64)
    dims: list = []

    def new_index(d):
        dims.append(d)
        return len(dims) - 1

    wire = [new_index(2) for _ in range(n)]
    raw: list = []

    def add(inds, data, p, core):
        raw.append(Tensor(list(inds), np.asarray(data, dtype=np.complex128), p, core, len(raw)))

    for q in range(n):
        add([wire[q]], [1.0, 0.0], (float(pos[q, 0]), float(pos[q, 1])), False)
    ltab = 0.0
    fcount = [0] * n
    for qs, U in circ.gates:
        if len(qs) == 1:
            q = qs[0]
            p = (float(pos[q, 0]), float(pos[q, 1]))
            if diag_hyper and _is_diag(U):
                add([wire[q]], np.diag(U), p, False)
            else:
                w = new_index(2)
                add([w, wire[q]], U, p, False)
                wire[q] = w
            continue
        a, b = qs
        fcount[a] += 1
        fcount[b] += 1
        xa, xb = pos[a], pos[b]
        dx, dy = float(xa[0] - xb[0]), float(xa[1] - xb[1])
        ltab = max(ltab, math.sqrt(dx * dx + dy * dy))
        pa = (float(xa[0] + (xb[0] - xa[0]) / 4.0), float(xa[1] + (xb[1] - xa[1]) / 4.0))
        pb = (float(xb[0] + (xa[0] - xb[0]) / 4.0), float(xb[1] + (xa[1] - xb[1]) / 4.0))
        diag = _is_diag(U)
        if diag and diag_hyper:
            add([wire[a], wire[b]], np.diag(U).reshape(2, 2), pb, True)
            continue
        if diag:
            s = new_index(2)
            wa = new_index(2)
            wb = new_index(2)
            X = np.zeros((2, 2, 2), np.complex128)
            Y = np.zeros((2, 2, 2), np.complex128)
            for i in range(2):
                X[i, i, i] = 1.0
                for k in range(2):
                    Y[i, i, k] = U[2 * k + i, 2 * k + i]
        else:
            s = new_index(4)
            wa = new_index(2)
            wb = new_index(2)
            X = np.zeros((2, 2, 4), np.complex128)
            Y = np.zeros((2, 2, 4), np.complex128)
            for i in range(2):
                for j in range(2):
                    X[i, j, 2 * i + j] = 1.0
                    for k in range(4):
                        Y[i, j, k] = U[2 * (k >> 1) + i, 2 * (k & 1) + j]
        add([wa, wire[a], s], X, pa, True)
        add([wb, wire[b], s], Y, pb, True)
        wire[a], wire[b] = wa, wb

    out_leg = list(wire)
    outs = set(out_leg)
    alive = [True] * len(raw)
    hold: dict = {}
    for t, T in enumerate(raw):
        for i in T.inds:
            hold.setdefault(i, set()).add(t)

    def others(idx, exclude):
        return [h for h in hold.get(idx, ()) if h not in exclude]

    # --- absorption (R2) ---
    changed = True
    while changed:
        changed = False
        for t in range(len(raw)):
            if not alive[t] or raw[t].core:
                continue
            T = raw[t]
            nbrs = sorted({h for i in T.inds for h in others(i, (t,))})
            if not nbrs:
                continue
            later = [h for h in nbrs if h > t]
            tgt = later[0] if later else nbrs[-1]
            keep = set()
            for i in set(T.inds) | set(raw[tgt].inds):
                if i in outs or others(i, (t, tgt)):
                    keep.add(i)
            inds, data = _pair_contract(raw[tgt], T, keep, None)
            for i in raw[tgt].inds:
                hold[i].discard(tgt)
            for i in T.inds:
                hold[i].discard(t)
            raw[tgt] = Tensor(inds, data, raw[tgt].pos, raw[tgt].core, raw[tgt].created)
            for i in inds:
                hold.setdefault(i, set()).add(tgt)
            alive[t] = False
            changed = True
    # promote isolated non-core tensors (qubits without two-qubit gates)
    for t in range(len(raw)):
        if alive[t] and not raw[t].core:
            q = next(q for q in range(n) if out_leg[q] in raw[t].inds)
            raw[t].core = True
            raw[t].pos = (float(pos[q, 0]), float(pos[q, 1]))
    # --- R4: sum out indices held by one tensor only ---
    for t in range(len(raw)):
        if not alive[t]:
            continue
        T = raw[t]
        for i in list(T.inds):
            if i not in outs and not others(i, (t,)):
                ax = T.inds.index(i)
                T.data = T.data.sum(axis=ax)
                T.inds.pop(ax)
                hold[i].discard(t)
    final = [raw[t] for t in range(len(raw)) if alive[t]]
    # canonical axis order: output legs first, then ascending index id
    for T in final:
        order = sorted(range(len(T.inds)), key=lambda a: (T.inds[a] not in outs, T.inds[a]))
        T.data = np.ascontiguousarray(np.transpose(T.data, order)) if T.inds else T.data
        T.inds = [T.inds[a] for a in order]
    out_owner = [next(k for k, T in enumerate(final) if out_leg[q] in T.inds) for q in range(n)]
    # sphere radius l/4 + eps (Theorem 2 proof), eps = eps_frac * r
    rmin = math.inf
    for i in range(n):
        for j in range(i + 1, n):
            dx, dy = float(pos[i, 0] - pos[j, 0]), float(pos[i, 1] - pos[j, 1])
            d = math.sqrt(dx * dx + dy * dy)
            rmin = min(rmin, d)
    if not math.isfinite(rmin) or rmin <= 0:
        rmin = 1.0
    radius = ltab / 4.0 + eps_frac * rmin
    F = max(fcount) if fcount else 0
    # k bound: only U (no U^dagger) -> F ((l/4 + r/4)/(r/4))^d, d = 2 (l.123)
    g = (ltab + rmin) / rmin
    k_bound = max(1.0, float(F) * (g * g))
    return Network(dims, final, out_leg, out_owner, radius, k_bound, n,
                   extras=dict(l=ltab, r=rmin, F=F, diag_hyper=diag_hyper))
