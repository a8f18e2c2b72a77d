"""The multi-rank path that bench.py runs, with 2 ranks on cuda:0 (-m gpu): slices of one
amplitude partitioned by dist.slice_block and summed by dist.allreduce_sum_ on CUDA
tensors (gloo backend: one GPU is reachable, the ranks never wait on each other's
kernels), the order found by rank 0 and imported by rank 1 (dist.shared_order), bitstrings partitioned by dist.block_range / dist.bitstring_steps; the
reduced results against the oracle."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2208_01498_b200 as tb
    from paper_2208_01498_b200 import dist as pdist
    from tn_inputs import lattice_cz, sycamore, random_bitstrings
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    out = {}
    # slices of one amplitude (the --config 2 / 4 path): complex64 sliced Sycamore-type
    # plan (3 sliced bits) and a complex128 lattice plan (4 sliced bits)
    for name, circ, dtype, tgt in (("syc", sycamore(6, 3), tb.TN_C64, 16), ("lat", lattice_cz(5, 5, 10, 2), tb.TN_C128, 12)):
        net = tb.Network.from_circuit(circ)
        # the order as bench.py gets it: rank 0 searches, rank 1 imports the broadcast
        order = pdist.shared_order(lambda: tb.Order(net, seed=0, max_log2_size=tgt),
                                   lambda st, sl, mf: tb.Order.from_steps(net, st, sl, mf), device=dev)
        plan = tb.Plan(net, order, dtype=dtype, device=0)
        x = random_bitstrings(circ.n, 1, 4)[0]
        n_sl = plan.info()["n_slices"]
        live = plan.contributing_slice_ids(x, 0, n_sl)
        mine = pdist.slice_block(live, world, rank)
        K = -(-len(live) // world)
        amp = torch.zeros(K, dtype=torch.complex128, device=dev)
        bits_dev = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
        st = torch.cuda.current_stream().cuda_stream
        for j, s in enumerate(mine):
            plan.contract_profiled(bits_dev.data_ptr(), s, s + 1, amp[j:j + 1].data_ptr(), st)
        torch.cuda.synchronize()
        pdist.allreduce_sum_(amp)
        out[name] = (complex(amp.sum().item()), mine, n_sl, len(live), order.steps(), order.slices(), list(x))
    # bitstrings (the configs 1 / 3 path)
    circ = lattice_cz(4, 4, 8, 1)
    net = tb.Network.from_circuit(circ)
    order = tb.Order(net, seed=0)
    plan = tb.Plan(net, order, dtype=tb.TN_C128, device=0)
    bits = random_bitstrings(circ.n, 7, 9)
    amps = pdist.amplitudes_by_bitstring(lambda b: plan.amplitudes(np.array([b]))[0], bits, device=dev)
    lo, hi = pdist.block_range(len(bits), world, rank)
    items = pdist.bitstring_steps(lambda r, n: plan.contributing_slice_ids(bits[r], 0, n), range(lo, hi), 100)
    out["bits"] = (amps, (lo, hi), items)
    q.put((rank, out))
    dist.destroy_process_group()


def test_two_ranks_on_one_gpu_gloo():
    import torch.multiprocessing as mp
    from tn_inputs import lattice_cz, sycamore, random_bitstrings
    from oracle.network import build_network
    from oracle.contract import contract_tree
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=900) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    circs = {"syc": (sycamore(6, 3), 1e-5), "lat": (lattice_cz(5, 5, 10, 2), 1e-10)}
    for name, (circ, tol) in circs.items():
        a0, m0, n_sl, n_live, steps, sl, x = res[0][name]
        a1, m1, *_ = res[1][name]
        assert n_sl > 1 and m0 and m1 and not set(m0) & set(m1) and len(m0) + len(m1) == n_live
        assert a0 == a1                                  # both ranks hold the reduced value
        on = build_network(circ)
        want = contract_tree(on, steps, x)               # the unsliced oracle amplitude
        assert abs(a0 - want) <= tol * max(abs(want), 2.0 ** (-circ.n / 2)), (name, a0, want)
    circ = lattice_cz(4, 4, 8, 1)
    bits = random_bitstrings(circ.n, 7, 9)
    on = build_network(circ)
    from oracle.ssa import find_order
    steps, _ = find_order(on, seed=0)
    want = np.array([contract_tree(on, steps, b) for b in bits])
    for r in (0, 1):
        amps, (lo, hi), items = res[r]["bits"]
        assert np.allclose(amps, want, atol=1e-10 * 2.0 ** (-circ.n / 2), rtol=1e-10)
        assert [i[0] for i in items] == list(range(lo, hi)) and all(s == 0 for _, s in items)
    assert res[0]["bits"][1][1] == res[1]["bits"][1][0]
