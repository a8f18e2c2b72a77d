"""The benched plans and the benched code path (-m gpu; VERDICT r1 "verify the benched
plans").

* tn_contract_profiled (the launcher bench.py times: a profiled CUDA graph with event records;
  eager launches with TN_PROFILE_GRAPH=0) is
  bit-identical to tn_contract_device (the CUDA-graph path) and accounts every flop;
* configs[1], [2], [4] at full size with the bench's kernels (K-slabs / row slabs, CTA
  pairs, persistent tiles, K-chunks at the 2^30-entry pack cap): one slice of an order at
  slicing target 2^31 through the complex64 plan and through the complex128 plan of the
  same order (the DMMA / fp64 path, oracle-verified at 1e-13 per step), agreeing to 1e-5
  of the RMS slice;
* one full configs[1] amplitude through the bench plan itself (2^32 slicing target, best
  of 256 hierarchies, 64 contributing slices, slice-invariant prologue) against the same
  amplitude through a differently sliced plan (2^34 target: other hierarchy, other
  slices, other slab structure, with TN_SLICE_REUSE=0: no prologue).
"""
import os
import subprocess
import sys
import textwrap

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tn_inputs import config_circuit, lattice_cz, sycamore, random_bitstrings

import paper_2208_01498_b200 as tb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


@pytest.mark.parametrize("dtype", [tb.TN_C64, tb.TN_C128])
def test_profiled_path_matches_graph_path(dtype):
    dev = _cuda()
    c = sycamore(6, 3)
    net = tb.Network.from_circuit(c)
    order = tb.Order(net, seed=0, max_log2_size=16)
    plan = tb.Plan(net, order, dtype=dtype)
    info = plan.info()
    assert info["n_slices"] >= 8
    if dtype == tb.TN_C64:
        assert info["n_steps_tc"] > 0
    x = random_bitstrings(c.n, 1, 3)[0]
    bits = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    st = torch.cuda.current_stream().cuda_stream
    ns = info["n_slices"]
    a_prof = torch.zeros(ns, dtype=torch.complex128, device=dev)
    a_graph = torch.zeros(ns, dtype=torch.complex128, device=dev)
    flops = 0.0
    for s in range(ns):
        p = plan.contract_profiled(bits.data_ptr(), s, s + 1, a_prof[s:s + 1].data_ptr(), st)
        plan.contract_device(bits.data_ptr(), s, s + 1, a_graph[s:s + 1].data_ptr(), st)
        flops += sum(d["flops"] for d in p["kernels"].values())
        assert p["ms_gemm"] + p["ms_pack"] + p["ms_small"] + p["ms_other"] > 0
    torch.cuda.synchronize()
    assert torch.equal(a_prof, a_graph)
    assert abs(flops - info["flops_per_slice"] * ns) <= 1e-12 * flops
    assert abs(a_graph.sum().item() - plan.contract(x)) <= 1e-12 * abs(a_graph.sum().item()) + 1e-300


def test_profiled_eager_path_matches_graph_path():
    """TN_PROFILE_GRAPH=0 (child process): the profiled launcher's eager fallback, the same
    checks as above in both dtypes."""
    import subprocess, sys
    code = ("import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')\n"
            "import test_gpu_bench_plans as T, paper_2208_01498_b200 as tb\n"
            "for dt in (tb.TN_C64, tb.TN_C128):\n    T.test_profiled_path_matches_graph_path(dt)\n"
            "print('ok')\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                       env=dict(os.environ, TN_PROFILE_GRAPH="0"), cwd=ROOT)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


_C64_VS_C128 = textwrap.dedent("""
    import sys; sys.path.insert(0, '.')
    import numpy as np, paper_2208_01498_b200 as tb
    from tn_inputs import config_circuit, random_bitstrings
    ci, tgt, n_seeds, dt = CI, TGT, NSEEDS, DT
    c = config_circuit(ci)
    net = tb.Network.from_circuit(c)
    o = tb.Order(net, seed=0, n_seeds=n_seeds, max_log2_size=tgt)
    p = tb.Plan(net, o, dtype=dt)
    x = random_bitstrings(c.n, 1, 1)[0]
    sid = p.contributing_slice_ids(x, 0, 1)[0]
    st = p.steps()
    kinds = sorted(set(int(v) for v in st[:, 0]))
    a = p.contract(x, sid, sid + 1)
    print(repr((sid, p.info()["slice_bits"], kinds, a.real, a.imag)))
""")


@pytest.mark.parametrize("ci", [1, 2, 4])
def test_full_size_slice_complex64_vs_complex128(ci):
    """One slice at slicing target 2^31 (best of 64 hierarchies) of configs[ci]: the
    complex64 tensor-core plan against the complex128 plan of the same order, each in its
    own process (plans of up to ~180 GB)."""
    _cuda()
    torch.cuda.empty_cache()           # the child plans need the whole device
    res = {}
    for dt in (tb.TN_C64, tb.TN_C128):
        code = _C64_VS_C128.replace("CI", str(ci)).replace("TGT", "31").replace("NSEEDS", "64").replace("DT", str(dt))
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=1200)
        assert r.returncode == 0, r.stdout + r.stderr
        res[dt] = eval(r.stdout.strip().splitlines()[-1])
    s64, b64, k64, *v64 = res[tb.TN_C64]
    s128, b128, k128, *v128 = res[tb.TN_C128]
    assert (s64, b64) == (s128, b128)
    assert tb.TN_PATH_TC in k64
    a64, a128 = complex(*v64), complex(*v128)
    scale = 2.0 ** (-config_circuit(ci).n / 2 - b64 / 2)          # RMS of one slice
    assert abs(a128) > 0
    rel = abs(a64 - a128) / max(abs(a128), scale)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "c64_vs_c128_slices.jsonl"), "a") as f:
        f.write(repr({"config": ci, "slice": s64, "slice_bits": b64, "c64": a64, "c128": a128, "rel": rel}) + "\n")
    assert rel <= 1e-5, (a64, a128, scale)


_FULL_AMP = textwrap.dedent("""
    import sys; sys.path.insert(0, '.')
    import numpy as np, paper_2208_01498_b200 as tb
    from tn_inputs import config_circuit, random_bitstrings
    c = config_circuit(1)
    net = tb.Network.from_circuit(c)
    o = tb.Order(net, seed=0, n_seeds=256, max_log2_size=TGT)
    p = tb.Plan(net, o, dtype=tb.TN_C64)
    x = random_bitstrings(c.n, 1024, 1)[0]          # the bench batch's first bitstring
    a = p.amplitudes(np.array([x]))[0]              # all slices (zero ones skipped)
    print(repr((p.info()["slice_bits"], p.contributing_slices(x), p.info()["flops_prologue"] > 0, a.real, a.imag)))
""")


def test_config1_full_amplitude_two_slicings():
    """A full configs[1] amplitude through the bench plan (2^32, slice reuse) and through a
    2^34 plan without slice reuse (TN_SLICE_REUSE=0)."""
    _cuda()
    torch.cuda.empty_cache()           # the child plans need the whole device
    import bench
    res = []
    for tgt, env in ((bench.SPEC[1]["slice_log"], {}), (34, {"TN_SLICE_REUSE": "0"})):
        r = subprocess.run([sys.executable, "-c", _FULL_AMP.replace("TGT", str(tgt))], capture_output=True, text=True,
                           cwd=ROOT, timeout=1800, env=dict(os.environ, **env))
        assert r.returncode == 0, r.stdout + r.stderr
        res.append(eval(r.stdout.strip().splitlines()[-1]))
    (b1, c1, pro1, *v1), (b2, c2, pro2, *v2) = res
    assert b1 == 8 and c1 == 64 and pro1 and b2 == 6 and c2 == 32 and not pro2
    a1, a2 = complex(*v1), complex(*v2)
    scale = 2.0 ** (-64 / 2)
    rel = abs(a1 - a2) / max(abs(a2), scale)
    with open(os.path.join(ROOT, "gpurun_out", "config1_full_amplitude.txt"), "w") as f:
        f.write(f"configs[1] <x|C|0> = {a1} (bench plan, 2^32 + reuse), {a2} (2^34, no reuse), rel diff {rel:.3e}\n")
    assert rel <= 1e-5, (a1, a2)


def test_slice_reuse_prologue():
    """Slice reuse: the slice-invariant prologue runs once per
    bitstring.  (a) plan.info reports a prologue and a frontier; (b) tn_prepare + the
    slices through tn_contract_prepared (graph and profiled) sum to the tn_contract_device
    amplitude and to the unsliced oracle; (c) a plan built with TN_SLICE_REUSE=0 (child
    process) gives bit-identical amplitudes through tn_amplitudes."""
    dev = _cuda()
    from oracle.network import build_network
    from oracle.contract import contract_tree
    c = lattice_cz(6, 6, 12, 8)
    net = tb.Network.from_circuit(c)
    order = tb.Order(net, seed=0, max_log2_size=19)
    plan = tb.Plan(net, order, dtype=tb.TN_C64)
    info = plan.info()
    assert info["n_slices"] >= 4 and info["flops_prologue"] > 0 and info["frontier_bytes"] > 0
    assert info["flops_prologue"] < info["flops_per_slice"]
    xs = random_bitstrings(c.n, 3, 6)
    st = torch.cuda.current_stream().cuda_stream
    on = build_network(c)
    ns = info["n_slices"]
    for x in xs:
        bits = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
        full = torch.zeros(1, dtype=torch.complex128, device=dev)
        plan.contract_device(bits.data_ptr(), 0, ns, full.data_ptr(), st)
        parts = torch.zeros(ns, dtype=torch.complex128, device=dev)
        plan.prepare(bits.data_ptr(), st)
        for s in range(ns):
            plan.contract_prepared(s, s + 1, parts[s:s + 1].data_ptr(), st, profiled=(s % 2 == 1))
        prof = torch.zeros(1, dtype=torch.complex128, device=dev)
        p = plan.prepare(bits.data_ptr(), st, profiled=True)
        assert abs(sum(d["flops"] for d in p["kernels"].values()) - info["flops_prologue"]) <= 1e-9 * info["flops_prologue"]
        plan.contract_prepared(0, ns, prof.data_ptr(), st)
        torch.cuda.synchronize()
        a_full, a_parts, a_prof = full.item(), parts.sum().item(), prof.item()
        # another contraction call invalidates the prepared bitstring
        plan.contract(x, 0, 1)
        with pytest.raises(tb.TnError):
            plan.contract_prepared(0, 1, prof.data_ptr(), st)
        assert abs(a_parts - a_full) <= 1e-12 * abs(a_full) and abs(a_prof - a_full) <= 1e-12 * abs(a_full)
        want = contract_tree(on, order.steps(), x)
        assert abs(a_full - want) <= 1e-5 * max(abs(want), 2.0 ** (-c.n / 2))
    code = textwrap.dedent("""
        import sys; sys.path.insert(0, '.')
        import numpy as np, paper_2208_01498_b200 as tb
        from tn_inputs import lattice_cz, random_bitstrings
        c = lattice_cz(6, 6, 12, 8)
        net = tb.Network.from_circuit(c)
        p = tb.Plan(net, tb.Order(net, seed=0, max_log2_size=19), dtype=tb.TN_C64)
        assert p.info()["flops_prologue"] == 0
        print(repr([complex(a) for a in p.amplitudes(random_bitstrings(c.n, 3, 6))]))
    """)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=600,
                       env=dict(os.environ, TN_SLICE_REUSE="0"))
    assert r.returncode == 0, r.stdout + r.stderr
    assert eval(r.stdout.strip().splitlines()[-1]) == [complex(a) for a in plan.amplitudes(xs)]


def test_deferred_profiling_matches_synchronous():
    """tn_profile_defer / tn_profile_collect (bench.py's timed region): a loop of deferred
    profiled slices gives the same amplitudes as the graph path, per-call algorithmic
    counters as in synchronous mode, and device times for every kernel class that ran
    (collected once at the end; a second collect returns nothing)."""
    dev = _cuda()
    c = sycamore(6, 3)
    net = tb.Network.from_circuit(c)
    plan = tb.Plan(net, tb.Order(net, seed=0, max_log2_size=16), dtype=tb.TN_C64)
    ns = plan.info()["n_slices"]
    x = random_bitstrings(c.n, 1, 5)[0]
    bits = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    st = torch.cuda.current_stream().cuda_stream
    a_sync = torch.zeros(ns, dtype=torch.complex128, device=dev)
    a_def = torch.zeros(ns, dtype=torch.complex128, device=dev)
    sync = [plan.contract_profiled(bits.data_ptr(), s, s + 1, a_sync[s:s + 1].data_ptr(), st) for s in range(ns)]
    plan.profile_defer(True)
    defer = [plan.contract_profiled(bits.data_ptr(), s, s + 1, a_def[s:s + 1].data_ptr(), st) for s in range(ns)]
    col = plan.profile_collect()
    plan.profile_defer(False)
    again = plan.profile_collect()
    torch.cuda.synchronize()
    assert torch.equal(a_sync, a_def)
    for p, q in zip(sync, defer):
        for name in p["kernels"]:
            assert p["kernels"][name]["flops"] == q["kernels"][name]["flops"]
            assert p["kernels"][name]["bytes"] == q["kernels"][name]["bytes"]
            assert q["kernels"][name]["ms"] == 0.0
    for name, d in col["kernels"].items():
        n_sync = sum(p["kernels"][name]["intervals"] for p in sync)
        assert d["intervals"] == n_sync, name
        assert (d["ms"] > 0) == (n_sync > 0), name
    assert all(d["intervals"] == 0 and d["ms"] == 0 for d in again["kernels"].values())


def test_deferred_profiling_with_prologue():
    """bench.py's timed loop on a plan with a slice-invariant prologue: tn_prepare and
    tn_contract_prepared with profiles in deferred mode over two bitstrings (both
    phases' profiled graphs alternate their two buffers) give bit-identical slice
    amplitudes to the unprofiled graph path, and the collected device times cover the
    prologue and every slice."""
    dev = _cuda()
    c = lattice_cz(6, 6, 12, 8)
    net = tb.Network.from_circuit(c)
    plan = tb.Plan(net, tb.Order(net, seed=0, max_log2_size=19), dtype=tb.TN_C64)
    info = plan.info()
    assert info["flops_prologue"] > 0
    ns = info["n_slices"]
    xs = random_bitstrings(c.n, 2, 8)
    st = torch.cuda.current_stream().cuda_stream
    want = torch.zeros(2 * ns, dtype=torch.complex128, device=dev)
    got = torch.zeros(2 * ns, dtype=torch.complex128, device=dev)
    bits = [torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in xs]
    for r in range(2):
        plan.prepare(bits[r].data_ptr(), st)
        for s in range(ns):
            plan.contract_prepared(s, s + 1, want[r * ns + s:r * ns + s + 1].data_ptr(), st)
    plan.profile_defer(True)
    flops = 0.0
    for r in range(2):
        p = plan.prepare(bits[r].data_ptr(), st, profiled=True)
        flops += sum(d["flops"] for d in p["kernels"].values())
        for s in range(ns):
            p = plan.contract_prepared(s, s + 1, got[r * ns + s:r * ns + s + 1].data_ptr(), st, profiled=True)
            flops += sum(d["flops"] for d in p["kernels"].values())
    col = plan.profile_collect()
    plan.profile_defer(False)
    torch.cuda.synchronize()
    assert torch.equal(want, got)
    expect = 2 * info["flops_prologue"] + 2 * ns * (info["flops_per_slice"] - info["flops_prologue"])
    assert abs(flops - expect) <= 1e-9 * expect
    assert col["ms_gemm"] > 0 and col["kernels"]["other"]["intervals"] == 2 * 1 + 2 * ns * 2
