"""Oracle pins (CPU, -m "not gpu").  Each test ties a piece of oracle/ to something
other than itself: brute force, closed forms, invariants, worked examples."""
import itertools
import json
import math
import os

import numpy as np
import pytest

from tn_inputs import Circuit, lattice_cz, sycamore, iqp, random3d, inverse_circuit, concat, random_bitstrings
from tn_inputs.circuits import haar_unitary
from oracle.network import build_network
from oracle import ssa
from oracle.ssa import find_order, step_costs, choose_slices, sliced_work
from oracle.contract import contract_tree, contract_pair, contract_pair_loops, kept_per_step, leaf_tensors
from oracle.statevector import statevector
from oracle import bounds
from oracle.rng import Stream, splitmix64

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def small_circuits():
    out = [lattice_cz(2, 3, 4, 11), lattice_cz(3, 3, 5, 12), iqp(3, 1, 13)]
    # generic U(4) gates (rank-4 split), nearest-neighbour on a 2x3 grid
    rng = np.random.default_rng(5)
    c = Circuit(6, np.array([(x, y) for y in range(2) for x in range(3)], dtype=float), name="u4")
    for t in range(4):
        for q in range(6):
            c.add((q,), haar_unitary(rng, 2))
        for a, b in ([(0, 1), (3, 4)], [(1, 2), (4, 5)], [(0, 3), (2, 5)], [(1, 4)])[t]:
            c.add((a, b), haar_unitary(rng, 4))
    out.append(c)
    # a qubit that never meets a two-qubit gate (promoted rank-1 tensor)
    c2 = lattice_cz(2, 2, 3, 14)
    c2.add((0,), haar_unitary(rng, 2))
    c3 = Circuit(5, np.vstack([c2.pos, [[5.0, 5.0]]]), name="idle")
    c3.gates = list(c2.gates) + [((4,), haar_unitary(rng, 2))]
    out.append(c3)
    # asymmetric diagonal two-qubit gates diag(e^{i phi_ab}) (R1's bond-2 split, R3's
    # hyperedge): CZ and controlled phases are symmetric in the two qubits, these are not,
    # so a split that swapped the qubits' roles would go unnoticed without them
    c4 = Circuit(6, np.array([(x, y) for y in range(2) for x in range(3)], dtype=float), name="diag_asym")
    for t in range(4):
        for q in range(6):
            c4.add((q,), haar_unitary(rng, 2))
        for a, b in ([(0, 1), (3, 4)], [(2, 1), (5, 4)], [(0, 3), (5, 2)], [(4, 1)])[t]:
            c4.add((a, b), np.diag(np.exp(1j * rng.uniform(0, 2 * np.pi, 4))))
    out.append(c4)
    return out


def load_golden(name):
    d = json.load(open(os.path.join(GOLDEN, name)))
    c = Circuit(d["n"], np.array(d["pos"], dtype=float), name=name)
    for g in d["gates"]:
        c.add(tuple(g["qubits"]), np.array(g["re"]) + 1j * np.array(g["im"]))
    return c, {k: complex(*v) for k, v in d["amplitudes"].items()}


# ------------------------------------------------------------------ rng -------
def test_splitmix64_reference_values():
    # SplitMix64 published reference: seed 0 stream -> first outputs of splitmix64(0), (golden increments)
    assert splitmix64(0) == 0xE220A8397B1DCDAF
    s = Stream(0, 0)
    a = [s.u64() for _ in range(3)]
    assert len(set(a)) == 3
    u = Stream(7, 3).uniform()
    assert 0.0 <= u < 1.0


# -------------------------------------------------------------- network -------
@pytest.mark.parametrize("name", ["bell.json", "ghz_cz.json"])
@pytest.mark.parametrize("hyper", [False, True])
def test_golden_worked_examples(name, hyper):
    c, amps = load_golden(name)
    net = build_network(c, diag_hyper=hyper)
    steps, _ = find_order(net, seed=3, n_seeds=1)
    for bits, want in amps.items():
        got = contract_tree(net, steps, [int(ch) for ch in bits])
        assert abs(got - want) < 1e-14, (bits, got, want)


@pytest.mark.parametrize("ci", range(6))
@pytest.mark.parametrize("hyper", [False, True])
def test_network_matches_statevector(ci, hyper):
    c = small_circuits()[ci]
    net = build_network(c, diag_hyper=hyper)
    steps, _ = find_order(net, seed=ci, n_seeds=1)
    psi = statevector(c)
    for bits in random_bitstrings(c.n, 6, ci):
        got = contract_tree(net, steps, bits)
        want = psi[tuple(bits)]
        assert abs(got - want) < 1e-12, (bits, got, want)


def test_tensor_count_theorem2():
    # n = 2 * (number of two-qubit gates) tensors after absorption (Theorem 2 proof, l.123)
    c = lattice_cz(3, 4, 6, 1)
    net = build_network(c)
    assert len(net.tensors) == 2 * c.n_two_qubit


def test_norm_invariant():
    # sum_x |<x|C|0>|^2 = 1 (unitarity), brute force over all bitstrings
    c = lattice_cz(2, 4, 5, 21)
    net = build_network(c)
    steps, _ = find_order(net, seed=1, n_seeds=1)
    tot = 0.0
    for x in itertools.product([0, 1], repeat=c.n):
        tot += abs(contract_tree(net, steps, x)) ** 2
    assert abs(tot - 1.0) < 1e-12


def test_c_then_cdagger_is_identity():
    c = lattice_cz(3, 3, 4, 31)
    cc = concat(c, inverse_circuit(c))
    net = build_network(cc)
    steps, _ = find_order(net, seed=2, n_seeds=1)
    assert abs(contract_tree(net, steps, [0] * c.n) - 1.0) < 1e-12
    assert abs(contract_tree(net, steps, [1] + [0] * (c.n - 1))) < 1e-12


def test_iqp_closed_form():
    # <x|H^n D H^n|0> = 2^-n sum_z (-1)^{x.z} exp(i phi(z))  with phi from the diagonal gates
    c = iqp(3, 1, 41)
    n = c.n
    phase = np.zeros(2 ** n, dtype=np.complex128)
    for z in range(2 ** n):
        zb = [(z >> (n - 1 - q)) & 1 for q in range(n)]
        p = 1.0 + 0j
        for qs, U in c.gates:
            if len(qs) == 1 and abs(U[0, 1]) == 0 and abs(U[1, 0]) == 0:
                p *= U[zb[qs[0]], zb[qs[0]]]
            elif len(qs) == 2:
                p *= U[2 * zb[qs[0]] + zb[qs[1]], 2 * zb[qs[0]] + zb[qs[1]]]
        phase[z] = p
    net = build_network(c, diag_hyper=True)
    steps, _ = find_order(net, seed=0, n_seeds=1)
    for x in random_bitstrings(n, 5, 4):
        want = 0j
        for z in range(2 ** n):
            zb = [(z >> (n - 1 - q)) & 1 for q in range(n)]
            want += (-1) ** sum(int(a) * b for a, b in zip(x, zb)) * phase[z]
        want /= 2 ** n
        assert abs(contract_tree(net, steps, x) - want) < 1e-12


def test_diag_hyper_shrinks_iqp_cut():
    # the hyperedge reading (R3) is what makes IQP tractable: same values, much smaller cost
    c = iqp(4, 2, 42)
    n1 = build_network(c, diag_hyper=False)
    n2 = build_network(c, diag_hyper=True)
    s1, _ = find_order(n1, seed=0, n_seeds=1)
    s2, _ = find_order(n2, seed=0, n_seeds=1)
    m1 = max(m for m, _ in step_costs(n1, s1))
    m2 = max(m for m, _ in step_costs(n2, s2))
    assert m2 < m1
    x = [0] * c.n
    assert abs(contract_tree(n1, s1, x) - contract_tree(n2, s2, x)) < 1e-12


# ------------------------------------------------------------- Eq. (3) --------
def test_eq3_operation_count_matches_executed():
    c = lattice_cz(2, 2, 3, 51)
    net = build_network(c)
    steps, _ = find_order(net, seed=0, n_seeds=1)
    sc = step_costs(net, steps)
    kept = kept_per_step(net, steps)
    n = len(net.tensors)
    nodes = dict(enumerate(leaf_tensors(net, [0, 1, 1, 0])))
    total_ops = 0
    for k, (a, b) in enumerate(steps):
        (Ai, A), (Bi, B) = nodes.pop(a), nodes.pop(b)
        kk, res, n_mul, n_add = contract_pair_loops(Ai, A, Bi, B, kept[k], net.dims)
        assert n_mul == 2 ** sc[k][0]          # M of Eq. (3) = executed multiplications
        assert n_add <= 2 ** sc[k][0]          # additions bounded by M
        total_ops += n_mul + n_add
        ref_inds, ref = contract_pair(Ai, A, Bi, B, kept[k], net.dims)
        assert sorted(kk) == ref_inds
        for key, v in res.items():
            idx = tuple(key[kk.index(i)] for i in ref_inds) if ref_inds else ()
            assert abs(ref[idx] - v) < 1e-13
        nodes[n + k] = (ref_inds, ref)
        assert sc[k][1] == sum(net.log2dim(i) for i in ref_inds)
    assert total_ops <= sum(2 * 2 ** m for m, _ in sc)     # t <= sum 2 M (Eq. 3)


def test_slicing_sums_to_unsliced():
    c = lattice_cz(3, 3, 6, 61)
    net = build_network(c)
    steps, _ = find_order(net, seed=0, n_seeds=1)
    big = max(r for _, r in step_costs(net, steps))
    sl = choose_slices(net, steps, big - 3)
    assert len(sl) >= 1
    x = random_bitstrings(c.n, 1, 3)[0]
    a = contract_tree(net, steps, x)
    b = contract_tree(net, steps, x, sliced=sl)
    assert abs(a - b) < 1e-12
    # every sliced-contraction tensor respects the size target
    kept = kept_per_step(net, steps)
    assert all(sum(net.log2dim(i) for i in kk if i not in sl) <= big - 3 for kk in kept)


def test_sliced_work_counts_executed_multiplications():
    """sliced_work (the R10 / R11 objective) = the multiplications a literal nested-loop
    execution (Eq. (3): M per step) performs over every slice of the sliced contraction;
    without slices it is half the Eq. (3) total sum_k 2 M_k."""
    c = lattice_cz(2, 3, 4, 62)
    net = build_network(c)
    steps, _ = find_order(net, seed=0, n_seeds=1)
    assert sliced_work(net, steps, []) == sum(2.0 ** m for m, _ in step_costs(net, steps))
    big = max(r for _, r in step_costs(net, steps))
    sl = choose_slices(net, steps, big - 2)
    assert len(sl) >= 1
    kept = kept_per_step(net, steps)
    x = random_bitstrings(c.n, 1, 4)[0]
    n = len(net.tensors)
    muls = 0
    for vals in itertools.product(*[range(net.dims[i]) for i in sl]):
        fixed = dict(zip(sl, vals))
        nodes = dict(enumerate(leaf_tensors(net, x, fixed)))
        for k, (a, b) in enumerate(steps):
            (Ai, A), (Bi, B) = nodes.pop(a), nodes.pop(b)
            kk = [i for i in kept[k] if i not in fixed]
            _, _, n_mul, _ = contract_pair_loops(Ai, A, Bi, B, kk, net.dims)
            muls += n_mul
            nodes[n + k] = contract_pair(Ai, A, Bi, B, kk, net.dims)
    assert sliced_work(net, steps, sl) == muls


def test_find_order_keeps_least_sliced_work():
    """R10 with a slicing target: the kept hierarchy has the smallest sliced work among
    the n_seeds candidates (each candidate = the n_seeds=1 hierarchy of its stream)."""
    c = lattice_cz(4, 4, 8, 63)
    net = build_network(c)
    tgt = 8
    steps, _ = find_order(net, seed=5, n_seeds=3, max_log2_size=tgt)
    w = sliced_work(net, steps, choose_slices(net, steps, tgt))
    cands = []
    for r in range(3):
        ctx = ssa._Ctx(net, 5, 8, 32, 64, 256)
        ssa._build(ctx, list(range(len(net.tensors))), 1 + r, 0)
        cands.append(sliced_work(net, ctx.steps, choose_slices(net, ctx.steps, tgt)))
    assert w == min(cands)


# ------------------------------------------------------------ geometry --------
def test_stereographic_projection_closed_forms():
    x, y, z = ssa.stereo(np.array([0.0, 1.0, 3.0]), np.array([0.0, 0.0, 4.0]))
    assert (x[0], y[0], z[0]) == (0.0, 0.0, -1.0)          # origin -> south pole
    assert (x[1], y[1], z[1]) == (1.0, 0.0, 0.0)           # unit circle -> equator
    assert abs(x[2] - 6 / 26) < 1e-15 and abs(y[2] - 8 / 26) < 1e-15 and abs(z[2] - 24 / 26) < 1e-15
    r = np.random.default_rng(0).normal(size=(2, 100)) * 5
    a, b, c = ssa.stereo(r[0], r[1])
    assert np.allclose(a * a + b * b + c * c, 1.0, atol=1e-14)


def test_rotation_to_pole():
    rng = np.random.default_rng(1)
    for _ in range(20):
        c = tuple(rng.normal(size=3) * 0.3)
        R, nc = ssa.rotation_to_pole(c)
        R = np.array(R)
        assert np.allclose(R @ R.T, np.eye(3), atol=1e-13)
        assert np.allclose(R @ np.array(c), [0, 0, np.linalg.norm(c)], atol=1e-13)


def _pi(q):
    s = q @ q
    return np.array([2 * q[0], 2 * q[1], s - 1]) / (s + 1)


def _pi_inv(z):
    return np.array([z[0], z[1]]) / (1 - z[2])


def test_separator_circle_matches_pointwise_map():
    """Step 6 closed form vs a literal pointwise evaluation of Pi^-1 o R^T o D_a^-1."""
    rng = np.random.default_rng(2)
    for _ in range(30):
        c = rng.normal(size=3)
        c = c / np.linalg.norm(c) * rng.uniform(0.05, 0.9)
        R, nc = ssa.rotation_to_pole(tuple(c))
        alpha = math.sqrt((1 - nc) / (1 + nc))
        u = rng.normal(size=3)
        u /= np.linalg.norm(u)
        sep = ssa.separator_circle(tuple(u), R, alpha)
        # points on the great circle C
        e1 = np.cross(u, [1.0, 0, 0] if abs(u[0]) < 0.9 else [0, 1.0, 0])
        e1 /= np.linalg.norm(e1)
        e2 = np.cross(u, e1)
        for th in np.linspace(0, 2 * np.pi, 13)[:-1]:
            z = math.cos(th) * e1 + math.sin(th) * e2
            if z[2] > 1 - 1e-6:
                continue
            w = _pi(_pi_inv(z) / alpha)               # D_alpha^{-1}
            w = np.array(R).T @ w                      # R^T
            if w[2] > 1 - 1e-9:
                continue
            p = _pi_inv(w)                             # Pi^{-1}
            if np.linalg.norm(p) > 1e6:
                continue
            if sep[0] == "circle":
                _, cx, cy, rho = sep
                assert abs(math.hypot(p[0] - cx, p[1] - cy) - rho) < 1e-7 * max(1.0, rho)
            else:
                _, b0, b1, C0, nb = sep
                assert abs(2 * (b0 * p[0] + b1 * p[1]) - C0) < 1e-7 * max(1, nb)


def test_centerpoint_of_regular_simplex_is_centroid():
    v = np.array([[1, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]], dtype=float) / math.sqrt(3)
    pts = np.repeat(v, 3, axis=0)          # 12 points, 3 copies of each vertex
    c = ssa.centerpoint(list(pts[:, 0]), list(pts[:, 1]), list(pts[:, 2]), Stream(0, 9))
    assert np.linalg.norm(c) < 1e-9


def test_centerpoint_brute_force_depth():
    """Every closed half-space containing c holds >= a/(d+2) - (boundary slack) of the
    sample: brute force over all planes through c and a pair of points."""
    rng = np.random.default_rng(3)
    for trial in range(5):
        P = rng.normal(size=(14, 3))
        P /= np.linalg.norm(P, axis=1)[:, None]
        c = np.array(ssa.centerpoint(list(P[:, 0]), list(P[:, 1]), list(P[:, 2]), Stream(trial, 1)))
        worst = 14
        for i in range(14):
            for j in range(i + 1, 14):
                nrm = np.cross(P[i] - c, P[j] - c)
                if np.linalg.norm(nrm) < 1e-9:
                    continue
                s = (P - c) @ nrm
                worst = min(worst, int((s >= -1e-9).sum()), int((s <= 1e-9).sum()))
        assert worst * 4 >= 14 - 4, worst       # (d+1+delta):1 depth with the 2-point slack


def test_order_is_a_binary_tree_and_deterministic():
    c = lattice_cz(4, 4, 8, 0)
    net = build_network(c)
    s1, _ = find_order(net, seed=5)
    s2, _ = find_order(net, seed=5)
    assert s1 == s2
    n = len(net.tensors)
    seen = set()
    for k, (a, b) in enumerate(s1):
        assert a not in seen and b not in seen and a < n + k and b < n + k
        seen.update((a, b))
    assert len(s1) == n - 1 and len(seen) == 2 * n - 2


def test_hierarchy_cost_below_theorem1_bound():
    c = lattice_cz(4, 4, 8, 0)
    net = build_network(c)
    steps, _ = find_order(net, seed=0)
    t = sum(2.0 * 2.0 ** m for m, _ in step_costs(net, steps))
    n = len(net.tensors)
    M = max(2 ** sum(net.log2dim(i) for i in net.closed_inds(k)) for k in range(n))
    assert math.log2(t) < bounds.theorem1_log2(n, M, net.k_bound)


def test_theorem_constants():
    assert abs(bounds.a_d(2) - (4 + 2 * math.sqrt(3))) < 1e-12
    assert abs(bounds.a2_prime() - 5.3705) < 1e-3 and bounds.a2_prime() < bounds.a_d(2)
    assert abs(1 / math.log2(1.5) - 1.7095112913514547) < 1e-12


# ------------------------------------------------------------ degenerate ------
def test_degenerate_circuits_closed_forms():
    """A single qubit, a product state, no gates, two disconnected components: the
    oracle's network + tree contraction equals the closed-form amplitude for every
    bitstring (tests/degenerate.py)."""
    from degenerate import degenerate_circuits, all_bitstrings
    from oracle.contract import contract_tree
    for c, amp in degenerate_circuits():
        on = build_network(c)
        steps, _ = ssa.find_order(on, seed=0)
        for x in all_bitstrings(c.n):
            want = amp(x)
            got = contract_tree(on, steps, x)
            assert abs(got - want) <= 1e-12, (c.name, x, got, want)
