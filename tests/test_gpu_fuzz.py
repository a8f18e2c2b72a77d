"""Randomized whole-plan parity (-m gpu): small circuits of every family, random slicing
targets (so slice reuse, provably zero slices, slabs and the gathering kernels all occur
in varied combinations), both dtypes, amplitudes through tn_amplitudes (one lane and two)
against the unsliced oracle along the same (bit-identical) order."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tn_inputs import lattice_cz, sycamore, iqp, random3d, random_bitstrings
from oracle.network import build_network
from oracle.ssa import find_order
from oracle.contract import contract_tree

import paper_2208_01498_b200 as tb


def _circuit(kind, seed):
    """big enough for tensor-core, skinny and wide steps (largest steps 2^21 .. 2^27)"""
    rng = np.random.default_rng(seed)
    if kind == "lattice":
        return lattice_cz(int(rng.integers(5, 7)), 6, int(rng.integers(10, 13)), seed), False
    if kind == "sycamore":
        return sycamore(int(rng.integers(5, 7)), seed), False
    if kind == "iqp":
        return iqp(int(rng.integers(6, 8)), 2, seed), True
    return random3d(7, int(rng.integers(8, 11)), seed, n_patches=1, patch=4), False


_SEEN = set()


@pytest.mark.parametrize("case", range(24))
def test_random_plans_match_oracle(case):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    kinds = ["lattice", "sycamore", "iqp", "random3d"]
    kind = kinds[case % 4]
    c, hyper = _circuit(kind, 1000 + case)
    on = build_network(c, diag_hyper=hyper)
    cn = tb.Network.from_circuit(c, diag_hyper=hyper)
    full = tb.Order(cn, seed=case)
    big = full.info()["max_size_log2"]
    rng = np.random.default_rng(case)
    tgt = int(max(4, big - int(rng.integers(2, 6)))) if case % 3 else 0      # every third unsliced
    co = tb.Order(cn, seed=case, max_log2_size=tgt)
    osteps, _ = find_order(on, seed=case, max_log2_size=tgt)
    assert co.steps() == osteps
    dtype = tb.TN_C128 if case % 2 else tb.TN_C64
    plan = tb.Plan(cn, co, dtype=dtype)
    st = plan.steps()
    _SEEN.update((int(p), dtype) for p in st[:, 0])
    if plan.info()["flops_prologue"] > 0:
        _SEEN.add(("reuse", dtype))
    bits = random_bitstrings(c.n, 3, case)
    got1 = plan.amplitudes(bits)
    plan.set_lanes(2)
    got2 = plan.amplitudes(bits)
    assert np.array_equal(got1, got2)
    tol = 1e-10 if dtype == tb.TN_C128 else 1e-5
    for x, g in zip(bits, got1):
        want = contract_tree(on, osteps, x)
        assert abs(g - want) <= tol * max(abs(want), 2.0 ** (-c.n / 2)), (kind, tgt, dtype, g, want)


def test_random_plans_covered_every_path():
    """the random plans above went through the small and tensor-core paths and slice reuse in
    both dtypes, and through the (gathering) wide kernel (skinny steps need larger circuits:
    configs[3]'s full-size plan test covers them)"""
    if not _SEEN:
        pytest.skip("random plans did not run")
    for dt in (tb.TN_C64, tb.TN_C128):
        for path in (tb.TN_PATH_SMALL, tb.TN_PATH_TC):
            assert (path, dt) in _SEEN, (path, dt, sorted(map(str, _SEEN)))
        assert ("reuse", dt) in _SEEN, dt
    assert any((tb.TN_PATH_WIDE, dt) in _SEEN for dt in (tb.TN_C64, tb.TN_C128))
