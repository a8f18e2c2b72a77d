"""C-ABI library, host side (CPU, -m "not gpu"): symbols, network construction and
the order/slicing search compared with the oracle -- bit-identical orders."""
import ctypes
import os
import re

import numpy as np
import pytest

from tn_inputs import config_circuit, lattice_cz, iqp, sycamore, random3d
from oracle.network import build_network
from oracle.ssa import find_order, choose_slices

import paper_2208_01498_b200 as tb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "tn.h")).read()
    declared = set(re.findall(r"\b(tn_[a-z0-9_]+)\s*\(", hdr))
    declared -= {"tn_network_s", "tn_order_s", "tn_plan_s"}
    lib = ctypes.CDLL(tb._lib.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert declared == set(tb.EXPORTED_SYMBOLS)


def test_errors_are_reported_not_fatal():
    with pytest.raises(tb.TnError, match="bad qubit"):
        tb.Network(2, np.zeros((2, 2)), np.array([[0, 5]], np.int32), np.zeros(16, np.complex128))
    with pytest.raises(tb.TnError):
        tb.Network(0, np.zeros((0, 2)), np.zeros((0, 2), np.int32), np.zeros(0, np.complex128))


def _compare_networks(c, hyper):
    on = build_network(c, diag_hyper=hyper)
    cn = tb.Network.from_circuit(c, diag_hyper=hyper)
    inf = cn.info()
    d, o = cn.dims()
    assert inf["n_tensors"] == len(on.tensors)
    assert list(d) == on.dims and list(o) == on.out_leg
    assert inf["radius"] == on.radius and inf["k_bound"] == on.k_bound
    for t, T in enumerate(on.tensors):
        inds, pos, data = cn.tensor(t)
        assert list(inds) == T.inds and tuple(pos) == T.pos
        assert np.max(np.abs(data - T.data)) <= 1e-13
    return on, cn


@pytest.mark.parametrize("ci", [0, 1, 2, 3, 4])
def test_network_identical_to_oracle(ci):
    _compare_networks(config_circuit(ci), hyper=(ci == 3))


@pytest.mark.parametrize("hyper", [False, True])
def test_network_identical_asymmetric_diagonal_gates(hyper):
    """Diagonal two-qubit gates that are not symmetric in their qubits (R1 bond-2 split,
    R3 hyperedge): the product's split must give each qubit its own role, as the oracle's
    (pinned to the state vector in tests/test_oracle.py) does."""
    from test_oracle import small_circuits
    c = [x for x in small_circuits() if x.name == "diag_asym"][0]
    _compare_networks(c, hyper)


@pytest.mark.parametrize("case", ["c0", "c3", "small_slice", "syc_small", "r3d_small"])
def test_order_and_slices_bit_identical(case):
    if case == "c0":
        c, hyper, seed, tgt = config_circuit(0), False, 11, 0
    elif case == "c3":
        c, hyper, seed, tgt = iqp(6, 2, 3), True, 5, 14
    elif case == "small_slice":
        c, hyper, seed, tgt = lattice_cz(5, 5, 8, 2), False, 3, 14
    elif case == "syc_small":
        c, hyper, seed, tgt = sycamore(4, 1), False, 2, 20
    else:
        c, hyper, seed, tgt = random3d(6, 6, 1, n_patches=1), False, 9, 16
    on, cn = _compare_networks(c, hyper)
    co = tb.Order(cn, seed=seed, max_log2_size=tgt)
    os_, _ = find_order(on, seed=seed, max_log2_size=tgt)
    assert co.steps() == os_
    if tgt:
        assert co.slices() == choose_slices(on, os_, tgt)


@pytest.mark.slow
def test_order_bit_identical_config1():
    c = config_circuit(1)
    on, cn = _compare_networks(c, False)
    co = tb.Order(cn, seed=7, max_log2_size=30)
    os_, _ = find_order(on, seed=7, max_log2_size=30)
    assert co.steps() == os_
    assert co.slices() == choose_slices(on, os_, 30)


def test_order_info_consistent():
    c = lattice_cz(4, 4, 8, 0)
    cn = tb.Network.from_circuit(c)
    o = tb.Order(cn, seed=1, max_log2_size=6)
    inf = o.info()
    assert inf["n_steps"] == cn.info()["n_tensors"] - 1
    assert inf["n_slice_assignments"] == 2 ** inf["n_slices"]
    assert inf["log2_slice_2M"] <= inf["log2_total_2M"] + 1e-9


def test_degenerate_networks_and_orders_identical():
    """Degenerate circuits (tests/degenerate.py: one qubit, product state, no gates,
    disconnected components): the C++ network and order equal the oracle's."""
    from degenerate import degenerate_circuits
    for c, _ in degenerate_circuits():
        on, cn = _compare_networks(c, False)
        co = tb.Order(cn, seed=0)
        os_, _ = find_order(on, seed=0)
        assert co.steps() == os_, c.name


@pytest.mark.parametrize("ci", [1, 2, 3, 4])
def test_bench_orders_bit_identical_to_oracle_files(ci):
    """The benched orders: tn_find_order with bench.py's SPEC (seed, hierarchies, slicing
    target) reproduces the order and the sliced indices the ORACLE found
    (oracle/orders/config<ci>.json, scripts/write_oracle_orders.py), and reports the same
    median fallbacks."""
    import json
    import bench
    path = os.path.join(ROOT, "oracle", "orders", f"config{ci}.json")
    o = json.load(open(path))
    spec = bench.SPEC[ci]
    assert (o["n_seeds"], o["max_log2_size"], o["diag_hyper"]) == (spec["n_seeds"], spec["slice_log"], spec["hyper"])
    cn = tb.Network.from_circuit(config_circuit(ci), diag_hyper=spec["hyper"])
    co = tb.Order(cn, seed=o["seed"], n_seeds=o["n_seeds"], max_log2_size=o["max_log2_size"])
    assert co.steps() == [tuple(p) for p in o["steps"]]
    assert co.slices() == o["slices"]
    assert co.info()["median_fallbacks"] == o["median_fallbacks"]


def test_order_import_roundtrip_and_validation():
    """tn_order_import: an order rebuilt from its steps and sliced indices has the same
    steps, slices and info (Eq. (3) costs recomputed); malformed trees and sliced
    indices are refused with TN_EINVAL (the handle is not created)."""
    c = lattice_cz(4, 4, 8, 2)
    net = tb.Network.from_circuit(c)
    o = tb.Order(net, seed=5, n_seeds=2, max_log2_size=6)
    st, sl = o.steps(), o.slices()
    assert len(sl) >= 1
    o2 = tb.Order.from_steps(net, st, list(reversed(sl)), o.info()["median_fallbacks"])
    assert o2.steps() == st and o2.slices() == sl and o2.info() == o.info()
    n = net.info()["n_tensors"]
    d, out = net.dims()
    bad_steps = [
        st[:-1],                                    # one step short: no single root
        [(st[0][0], st[0][0])] + st[1:],            # a node contracted with itself
        [(st[0][0], n + 5)] + st[1:],               # a node not yet created
        st[:1] + [(st[0][0], st[1][1])] + st[2:],   # a consumed node reused
        [(-1, st[0][1])] + st[1:],
    ]
    for bs in bad_steps:
        with pytest.raises(tb.TnError, match="tn_order_import"):
            tb.Order.from_steps(net, bs, sl)
    for bsl in ([sl[0], sl[0]], [len(d)], [-1], [int(out[0])]):
        with pytest.raises(tb.TnError, match="tn_order_import"):
            tb.Order.from_steps(net, st, bsl)
