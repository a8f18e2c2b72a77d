"""The benched plans and the benched code path (-m gpu; VERDICT r1 "verify the benched
plans").

* tn_contract_profiled (the launcher bench.py times: eager launches with CUDA events) is
  bit-identical to tn_contract_device (the CUDA-graph path) and accounts every flop;
* configs[1], [2], [4] at full size with the bench's kernels (K-slabs / row slabs, CTA
  pairs, persistent tiles, K-chunks at the 2^30-entry pack cap): one slice of an order at
  slicing target 2^31 through the complex64 plan and through the complex128 plan of the
  same order (the DMMA / fp64 path, oracle-verified at 1e-13 per step), agreeing to 1e-5
  of the RMS slice;
* one full configs[1] amplitude through the bench plan itself (2^34 slicing target, best
  of 256 hierarchies, 32 contributing slices) against the same amplitude through a
  differently sliced plan (2^33 target: other hierarchy, other slices, other slab
  structure).
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
    print(repr((p.info()["slice_bits"], p.contributing_slices(x), a.real, a.imag)))
""")


def test_config1_full_amplitude_two_slicings():
    """A full configs[1] amplitude through the bench plan (2^34) and through a 2^33 plan."""
    _cuda()
    res = []
    for tgt in (34, 33):
        r = subprocess.run([sys.executable, "-c", _FULL_AMP.replace("TGT", str(tgt))], capture_output=True, text=True,
                           cwd=ROOT, timeout=1800)
        assert r.returncode == 0, r.stdout + r.stderr
        res.append(eval(r.stdout.strip().splitlines()[-1]))
    (b34, c34, *v34), (b33, c33, *v33) = res
    assert b34 == 6 and c34 == 32 and b33 > b34
    a34, a33 = complex(*v34), complex(*v33)
    scale = 2.0 ** (-64 / 2)
    assert abs(a34 - a33) <= 1e-5 * max(abs(a33), scale), (a34, a33)
    print(f"configs[1] <x|C|0> = {a34} (2^34 plan), {a33} (2^33 plan)")
