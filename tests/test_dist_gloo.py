"""Multi-rank host logic with world_size 2 on gloo (CPU): slice partitioning + one
all-reduce, bitstring partitioning; the per-rank contraction is the oracle's sliced
contraction so the summed result must equal the serial amplitude."""
import itertools
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2208_01498_b200.dist import block_range, sliced_amplitude, amplitudes_by_bitstring


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from tn_inputs import lattice_cz, random_bitstrings
    from oracle.network import build_network
    from oracle.ssa import find_order, choose_slices
    from oracle.contract import contract_tree
    c = lattice_cz(3, 4, 6, 3)
    net = build_network(c)
    steps, _ = find_order(net, seed=1, n_seeds=1)
    sl = choose_slices(net, steps, 5)
    assigns = list(itertools.product(*[range(net.dims[i]) for i in sl]))
    x = random_bitstrings(c.n, 1, 2)[0]

    def contract_range(lo, hi):
        tot = 0j
        for vals in assigns[lo:hi]:
            # one slice: fix the sliced indices by restricting the oracle to one assignment
            tot += _one_slice(net, steps, x, sl, vals)
        return tot

    amp = sliced_amplitude(contract_range, len(assigns))
    bits = random_bitstrings(c.n, 5, 7)
    amps = amplitudes_by_bitstring(lambda b: contract_tree(net, steps, b), bits)
    if rank == 0:
        q.put((amp, contract_tree(net, steps, x), amps, [contract_tree(net, steps, b) for b in bits], len(sl)))
    dist.destroy_process_group()


def _one_slice(net, steps, x, sl, vals):
    from oracle.contract import kept_per_step, leaf_tensors, contract_pair
    kept = kept_per_step(net, steps)
    fixed = dict(zip(sl, vals))
    n = len(net.tensors)
    nodes = dict(enumerate(leaf_tensors(net, x, fixed)))
    for k, (a, b) in enumerate(steps):
        (Ai, A), (Bi, B) = nodes.pop(a), nodes.pop(b)
        nodes[n + k] = contract_pair(Ai, A, Bi, B, [i for i in kept[k] if i not in fixed], net.dims)
    v = 1 + 0j
    for _, d in nodes.values():
        v *= complex(d)
    return v


def test_block_range_partitions():
    for n in (0, 1, 7, 16, 1025):
        for w in (1, 2, 3, 8):
            got = [block_range(n, w, r) for r in range(w)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(got[i][1] == got[i + 1][0] for i in range(w - 1))
            assert max(h - l for l, h in got) - min(h - l for l, h in got) <= 1


def test_two_ranks_gloo_slices_and_bitstrings():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    amp, want, amps, wants, n_sl = q.get(timeout=600)
    for p in procs:
        p.join(timeout=60)
    assert n_sl >= 1
    assert abs(amp - want) < 1e-12
    assert np.allclose(amps, wants, atol=1e-12)


def test_slice_block_and_bitstring_steps():
    """bench.py's partition: slice blocks are disjoint, contiguous and cover the list;
    bitstring steps walk the rows in order, one contributing slice per step, no repeats."""
    from paper_2208_01498_b200.dist import slice_block, bitstring_steps
    live = [3, 5, 8, 13, 21, 34, 55]
    for w in (1, 2, 3, 8):
        blocks = [slice_block(live, w, r) for r in range(w)]
        assert sum(blocks, []) == live
    contrib = {0: [0, 2, 4], 1: [1], 2: [0, 1, 2, 3]}
    items = bitstring_steps(lambda r, n: contrib[r][:n], [0, 1, 2], 6)
    assert items == [(0, 0), (0, 2), (0, 4), (1, 1), (2, 0), (2, 1)]
    assert len(set(items)) == len(items)
    assert bitstring_steps(lambda r, n: contrib[r][:n], [1], 5) == [(1, 1)]


def _order_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2208_01498_b200 as tb
    from paper_2208_01498_b200.dist import shared_order
    from tn_inputs import sycamore
    from oracle.network import build_network
    from oracle.ssa import find_order, choose_slices
    c = sycamore(4, 3, 4, 5)
    net = tb.Network.from_circuit(c)
    calls = []

    def find():
        calls.append(rank)
        return tb.Order(net, seed=3, n_seeds=2, max_log2_size=4)

    o = shared_order(find, lambda st, sl, mf: tb.Order.from_steps(net, st, sl, mf))
    on = build_network(c)
    steps, _ = find_order(on, seed=3, n_seeds=2, max_log2_size=4)
    q.put((rank, calls, o.steps(), o.slices(), o.info(), steps, choose_slices(on, steps, 4)))
    dist.destroy_process_group()


def test_two_ranks_gloo_shared_order():
    """dist.shared_order (bench.py under torchrun): rank 0 alone runs the order search,
    rank 1 imports the broadcast steps and sliced indices (tn_order_import) -- both hold
    the oracle's order and slices, with the same order info."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_order_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=600) for _ in range(2)], key=lambda g: g[0])
    for p in procs:
        p.join(timeout=60)
    (r0, calls0, st0, sl0, inf0, osteps, oslices), (r1, calls1, st1, sl1, inf1, _, _) = got
    assert calls0 == [0] and calls1 == []
    assert st0 == st1 == osteps and sl0 == sl1 == oslices and len(sl0) >= 1
    assert inf0 == inf1
