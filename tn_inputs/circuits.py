"""Seeded circuit generators for the five BASELINE.json configs.

Conventions (shared by every consumer):
  * qubit q sits at pos[q] = (x, y) in R^2 (the d = 2 embedding of Theorem 2,
    PAPER.md l.115-125);
  * gates are applied in list order; a gate is (qubits, U) with qubits = (a,) and
    U a 2x2 complex matrix, or qubits = (a, b) and U a 4x4 complex matrix in the
    basis |x_a x_b>, index 2*x_a + x_b (x_a is the high bit);
  * the amplitude of bitstring x (x[q] in {0,1}) is <x|C|0...0>.

Random draws use numpy's PCG64 seeded per circuit; this is input generation only.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Circuit:
    n: int
    pos: np.ndarray                      # (n, 2) float64
    gates: list = field(default_factory=list)   # [(tuple qubits, ndarray U)]
    name: str = ""

    def add(self, qubits, U):
        U = np.asarray(U, dtype=np.complex128)
        assert U.shape == ((2, 2) if len(qubits) == 1 else (4, 4))
        self.gates.append((tuple(int(q) for q in qubits), U))

    @property
    def n_two_qubit(self):
        return sum(1 for q, _ in self.gates if len(q) == 2)

    def flat(self):
        """Flat arrays for the C-ABI: gate_qubits (G,2) int32 (-1 for 1q),
        gate_mats: concatenated row-major complex128 matrices (4 or 16 entries)."""
        G = len(self.gates)
        gq = np.full((G, 2), -1, dtype=np.int32)
        mats = []
        for i, (q, U) in enumerate(self.gates):
            gq[i, :len(q)] = q
            mats.append(U.reshape(-1))
        m = np.concatenate(mats) if mats else np.zeros(0, np.complex128)
        return (np.ascontiguousarray(self.pos, dtype=np.float64), gq,
                np.ascontiguousarray(m, dtype=np.complex128))


def haar_unitary(rng: np.random.Generator, d: int) -> np.ndarray:
    """Haar-random U(d) via QR of a complex Ginibre matrix with phase fix."""
    z = (rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))) / math.sqrt(2.0)
    q, r = np.linalg.qr(z)
    ph = np.diag(r) / np.abs(np.diag(r))
    return q * ph[None, :]


CZ = np.diag([1, 1, 1, -1]).astype(np.complex128)
H = np.array([[1, 1], [1, -1]], dtype=np.complex128) / math.sqrt(2.0)


def _grid_pos(rows, cols):
    return np.array([(c, r) for r in range(rows) for c in range(cols)], dtype=np.float64)


def _brickwork_patterns(rows, cols):
    """Four edge classes of the square lattice, each a matching:
    A horizontal bonds with even left column, B odd left column,
    C vertical bonds with even top row, D odd top row.  Applied in the
    alternating order A, C, B, D (horizontal / vertical alternate)."""
    q = lambda r, c: r * cols + c
    A = [(q(r, c), q(r, c + 1)) for r in range(rows) for c in range(0, cols - 1, 2)]
    B = [(q(r, c), q(r, c + 1)) for r in range(rows) for c in range(1, cols - 1, 2)]
    C = [(q(r, c), q(r + 1, c)) for r in range(0, rows - 1, 2) for c in range(cols)]
    D = [(q(r, c), q(r + 1, c)) for r in range(1, rows - 1, 2) for c in range(cols)]
    return [A, C, B, D]


def lattice_cz(rows: int, cols: int, depth: int, seed: int) -> Circuit:
    """configs[0]/[1]: each layer = Haar U(2) on every qubit, then CZ on the
    nearest-neighbour pairs of one of four alternating brickwork patterns."""
    rng = np.random.default_rng([seed, 0xC2])
    c = Circuit(rows * cols, _grid_pos(rows, cols), name=f"lattice_cz_{rows}x{cols}_d{depth}_s{seed}")
    pats = _brickwork_patterns(rows, cols)
    for t in range(depth):
        for qb in range(c.n):
            c.add((qb,), haar_unitary(rng, 2))
        for a, b in pats[t % 4]:
            c.add((a, b), CZ)
    return c


# --- Sycamore-type (configs[2]) -------------------------------------------------
SQRT_X = np.array([[1, -1j], [-1j, 1]], dtype=np.complex128) / math.sqrt(2.0)
SQRT_Y = np.array([[1, -1], [1, 1]], dtype=np.complex128) / math.sqrt(2.0)
SQRT_W = np.array([[1, -np.sqrt(1j)], [np.sqrt(-1j), 1]], dtype=np.complex128) / math.sqrt(2.0)


def fsim(theta: float, phi: float) -> np.ndarray:
    c, s = math.cos(theta), math.sin(theta)
    return np.array([[1, 0, 0, 0], [0, c, -1j * s, 0], [0, -1j * s, c, 0],
                     [0, 0, 0, np.exp(-1j * phi)]], dtype=np.complex128)


def sycamore(cycles: int, seed: int, rows: int = 9, per_row: int = 6, drop: int = 3) -> Circuit:
    """53 qubits: a 6x9 rotated square lattice (row y has qubits at x = 2k + (y mod 2))
    with one site removed; couplers join (x, y)-(x +- 1, y + 1) (diagonal couplings).
    Coupler classes: A = (+1, even y), B = (+1, odd y), C = (-1, even y), D = (-1, odd y);
    each class is a matching.  Cycle sequence A B C D C D A B repeated.  Every cycle
    applies one of {sqrt X, sqrt Y, sqrt W} to every qubit (never the same gate twice in
    a row on a qubit), then fSim(pi/2, pi/6) on the active class.  A final layer of
    single-qubit gates closes the circuit."""
    rng = np.random.default_rng([seed, 0x5C])
    sites = [(2 * k + (y % 2), y) for y in range(rows) for k in range(per_row)]
    del sites[drop]
    idx = {s: i for i, s in enumerate(sites)}
    c = Circuit(len(sites), np.array(sites, dtype=np.float64), name=f"sycamore_m{cycles}_s{seed}")
    classes = {}
    for (x, y), i in idx.items():
        for dx, cls_even, cls_odd in ((+1, "A", "B"), (-1, "C", "D")):
            j = idx.get((x + dx, y + 1))
            if j is not None:
                classes.setdefault(cls_even if y % 2 == 0 else cls_odd, []).append((i, j))
    seq = "ABCDCDAB"
    sq = [SQRT_X, SQRT_Y, SQRT_W]
    last = [-1] * c.n
    F = fsim(math.pi / 2, math.pi / 6)

    def layer_1q():
        for qb in range(c.n):
            choices = [g for g in range(3) if g != last[qb]]
            g = choices[int(rng.integers(len(choices)))]
            last[qb] = g
            c.add((qb,), sq[g])

    for m in range(cycles):
        layer_1q()
        for a, b in sorted(classes.get(seq[m % 8], [])):
            c.add((a, b), F)
    layer_1q()
    return c


# --- IQP (configs[3]) -------------------------------------------------------------
def iqp(L: int, radius: int, seed: int) -> Circuit:
    """Hadamard layer; Z-rotations diag(1, e^{i theta}) on every qubit; controlled-phase
    diag(1,1,1,e^{i phi}) on every pair within Chebyshev distance <= radius (angles
    uniform in [0, 2 pi)); final Hadamard layer."""
    rng = np.random.default_rng([seed, 0x19])
    c = Circuit(L * L, _grid_pos(L, L), name=f"iqp_{L}x{L}_r{radius}_s{seed}")
    for qb in range(c.n):
        c.add((qb,), H)
    for qb in range(c.n):
        th = rng.uniform(0, 2 * math.pi)
        c.add((qb,), np.diag([1, np.exp(1j * th)]))
    for a in range(c.n):
        ra, ca = divmod(a, L)
        for b in range(a + 1, c.n):
            rb, cb = divmod(b, L)
            if max(abs(ra - rb), abs(ca - cb)) <= radius:
                ph = rng.uniform(0, 2 * math.pi)
                c.add((a, b), np.diag([1, 1, 1, np.exp(1j * ph)]))
    for qb in range(c.n):
        c.add((qb,), H)
    return c


# --- non-homogeneous (2+1)D random circuit (configs[4]) --------------------------
def random3d(L: int, depth: int, seed: int, n_patches: int = 3, patch: int = 4,
             p_sparse: float = 0.3) -> Circuit:
    """Haar U(2) on every qubit each layer; two-qubit Haar U(4) gates on the brickwork
    pattern of the layer: always inside dense patch x patch patches (seeded,
    non-overlapping), with probability p_sparse elsewhere."""
    rng = np.random.default_rng([seed, 0x3D])
    c = Circuit(L * L, _grid_pos(L, L), name=f"random3d_{L}x{L}_d{depth}_s{seed}")
    dense = np.zeros((L, L), dtype=bool)
    placed = 0
    while placed < n_patches:
        r0, c0 = (int(v) for v in rng.integers(0, L - patch + 1, size=2))
        if dense[max(r0 - 1, 0):r0 + patch + 1, max(c0 - 1, 0):c0 + patch + 1].any():
            continue
        dense[r0:r0 + patch, c0:c0 + patch] = True
        placed += 1
    pats = _brickwork_patterns(L, L)
    for t in range(depth):
        for qb in range(c.n):
            c.add((qb,), haar_unitary(rng, 2))
        for a, b in pats[t % 4]:
            ina = dense[a // L, a % L] and dense[b // L, b % L]
            u = rng.uniform()
            if ina or u < p_sparse:
                c.add((a, b), haar_unitary(rng, 4))
    return c


def inverse_circuit(c: Circuit) -> Circuit:
    out = Circuit(c.n, c.pos.copy(), name=c.name + "_dag")
    for q, U in reversed(c.gates):
        out.add(q, U.conj().T)
    return out


def concat(c1: Circuit, c2: Circuit) -> Circuit:
    assert c1.n == c2.n
    out = Circuit(c1.n, c1.pos.copy(), name=c1.name + "+" + c2.name)
    out.gates = list(c1.gates) + list(c2.gates)
    return out


def random_bitstrings(n: int, count: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng([seed, 0xB1])
    return rng.integers(0, 2, size=(count, n), dtype=np.uint8)


# configs as listed in BASELINE.json (index -> (builder, dtype, n_bitstrings))
CONFIGS = {
    0: dict(name="lattice_cz_4x4_d8", build=lambda s=0: lattice_cz(4, 4, 8, s), dtype="c128", n_bitstrings=16),
    1: dict(name="lattice_cz_8x8_d16", build=lambda s=1: lattice_cz(8, 8, 16, s), dtype="c64", n_bitstrings=1024),
    2: dict(name="sycamore53_m14", build=lambda s=2: sycamore(14, s), dtype="c64", n_bitstrings=0),
    3: dict(name="iqp_10x10_r2", build=lambda s=3: iqp(10, 2, s), dtype="c128", n_bitstrings=256),
    4: dict(name="random3d_12x12_d20", build=lambda s=4: random3d(12, 20, s), dtype="c64", n_bitstrings=0),
}


def config_circuit(i: int, seed: int | None = None) -> Circuit:
    cfg = CONFIGS[i]
    return cfg["build"]() if seed is None else cfg["build"](seed)
