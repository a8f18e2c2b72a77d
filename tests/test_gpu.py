"""GPU parity tests (-m gpu): the CUDA path through the C ABI against the oracle.

Tolerances:
  * step level, complex128 (CUDA-core DFMA): |C - C_ref| <= 1e-12 * sum_k |A||B|
  * step level, complex64 (block-scaled fp16x2 tensor cores / fp32 FMA):
        |C - C_ref| <= (4 + 2 sqrt(K)) 2^-24 * sum_k |A||B|
    (fp32 storage of A and B: 2 x 2^-24 per product; the fp16x2 split represents each
    scaled element to <= 2^-24 |x| + 2^-38 max|chunk| and drops x1 y1 <= 2^-24 |x y|;
    sequential fp32 accumulation over K terms: a random walk of ~sqrt(K) roundings of
    2^-24, with a factor 2 margin)
  * amplitudes: complex128 |a - a_ref| <= 1e-10 * max(|a_ref|, 2^{-n/2});
    complex64 |a - a_ref| <= 1e-5 * max(|a_ref|, 2^{-n/2})  (BASELINE north_star, with the
    RMS amplitude 2^{-n/2} as the scale for amplitudes near zero)
"""
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tn_inputs import config_circuit, lattice_cz, iqp, sycamore, random_bitstrings, concat, inverse_circuit
from oracle.network import build_network
from oracle.ssa import find_order, choose_slices
from oracle.contract import contract_tree, contract_slice, contract_pair as oracle_pair

import paper_2208_01498_b200 as tb


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _rand(shape, seed, dtype):
    g = np.random.default_rng(seed)
    x = (g.standard_normal(shape) + 1j * g.standard_normal(shape)) / math.sqrt(2)
    return x.astype(np.complex64 if dtype == tb.TN_C64 else np.complex128)


def c64_tol(K):
    return (4.0 + 2.0 * math.sqrt(K)) * 2.0 ** -24


def tc_tol(K):
    """Step bound of the complex64 tensor-core path, relative to
    sum_k |A||B|: 12 units of 2^-24 for one 128-element chunk (fp32 storage of A and B,
    the fp16x2 split, the debiased truncating TMEM accumulation of T <= 48 MMA updates,
    the fp32 store of C) plus a random walk of round-to-nearest fp32 additions over the
    K / 128 promoted chunks."""
    return (12.0 + 2.0 * math.sqrt(max(K / 128.0, 1.0))) * 2.0 ** -24


def _run_pair(inds_a, inds_b, inds_c, dims, dtype, path, seed=0, gen=None):
    dev = _cuda()
    sa = [dims[i] for i in inds_a]
    sb = [dims[i] for i in inds_b]
    sc = [dims[i] for i in inds_c]
    gen = gen or _rand
    A = gen(sa, seed, dtype)
    B = gen(sb, seed + 1, dtype)
    tdt = torch.complex64 if dtype == tb.TN_C64 else torch.complex128
    tA = torch.from_numpy(A).to(dev)
    tB = torch.from_numpy(B).to(dev)
    tC = torch.full(sc, float("nan"), dtype=tdt, device=dev)
    torch.cuda.synchronize()
    tb.contract_pair(dtype, tA.data_ptr(), inds_a, tB.data_ptr(), inds_b, tC.data_ptr(), inds_c, dims, path)
    torch.cuda.synchronize()
    got = tC.cpu().numpy()
    ref_inds, ref = oracle_pair(list(inds_a), A.astype(np.complex128), list(inds_b), B.astype(np.complex128),
                                inds_c, dims)
    _, bound = oracle_pair(list(inds_a), np.abs(A).astype(np.complex128), list(inds_b),
                           np.abs(B).astype(np.complex128), inds_c, dims)
    perm = [ref_inds.index(i) for i in inds_c]
    ref = np.transpose(ref, perm) if perm else ref
    bound = np.abs(np.transpose(bound, perm) if perm else bound)
    return got, ref, bound


PAIR_CASES = [
    # (inds_a, inds_b, inds_c, dims) -- index ids are positions in dims
    ([0, 1], [1, 2], [0, 2], [2, 2, 2]),                                  # 2x2 matrix product
    ([0, 1, 2], [2, 3, 1], [0, 3], [2, 4, 2, 2]),                          # two contracted, dim 4
    ([0, 1, 2], [0, 2, 3], [0, 1, 3], [2, 2, 2, 2]),                       # batch (hyperedge) index
    ([3, 0, 1, 2], [4, 2, 1], [0, 3, 4], [2, 2, 2, 2, 2]),                 # permuted operand layouts
    ([0], [1], [0, 1], [2, 2]),                                            # outer product
    ([0, 1], [0, 1], [], [2, 4]),                                          # full contraction to a scalar
    (list(range(12)), list(range(12))[::-1], [], [2] * 12),                # K = 4096 -> one CTA per output
    ([0, 1] + list(range(2, 10)), list(range(2, 10)) + [10], [0, 1, 10], [2] * 11),  # K = 256 -> warp per output
]


@pytest.mark.parametrize("dtype", [tb.TN_C64, tb.TN_C128])
@pytest.mark.parametrize("case", range(len(PAIR_CASES)))
def test_pair_small_path(case, dtype):
    ia, ib, ic, dims = PAIR_CASES[case]
    got, ref, bound = _run_pair(ia, ib, ic, dims, dtype, tb.TN_PATH_SMALL, seed=case)
    K = int(np.prod([dims[i] for i in ia if i in ib and i not in ic])) if ia else 1
    tol = c64_tol(K) if dtype == tb.TN_C64 else 1e-12
    assert np.all(np.abs(got - ref) <= tol * bound + 1e-30)


def _gemm_case(nb, m, n, k, perm_seed=None):
    """indices: batch b0.., rows m.., cols n.., contracted k.. each of dim 2."""
    ids = list(range(nb + m + n + k))
    bt, mm, nn, kk = ids[:nb], ids[nb:nb + m], ids[nb + m:nb + m + n], ids[nb + m + n:]
    ia = bt + mm + kk
    ib = bt + kk + nn
    if perm_seed is not None:
        g = np.random.default_rng(perm_seed)
        ia = list(g.permutation(ia))
        ib = list(g.permutation(ib))
    return ia, ib, bt + mm + nn, [2] * len(ids)


TC_CASES = [
    (0, 7, 7, 4, None),       # exactly one 128x128 tile, K = 16
    (0, 6, 5, 4, None),       # ragged: M = 64 < 128, N = 32 < BN
    (0, 9, 3, 10, 12),        # skinny N = 8 (one eighth of a 64-wide tile), permuted
    (0, 9, 8, 9, None),       # 4 x 2 tiles, K = 512 (16 stages)
    (2, 7, 6, 5, 3),          # batch 4, permuted layouts folded into the pack
    (0, 10, 10, 12, 5),       # several tiles, K = 4096, permuted
    (0, 7, 8, 14, None),      # K = 16384: split-K over 4 CTAs + fp64 reduction
    (1, 6, 7, 13, 7),         # split-K with batch and ragged M
    # M >= 256 and N >= 128: CTA-pair kernel (cta_group::2, 256 x 128 tiles)
    (0, 8, 7, 4, None),       # one pair tile, K = 16
    (2, 8, 7, 10, 3),         # batch 4, permuted, 32 stages
    (0, 9, 9, 14, 11),        # 2 x 4 pair tiles, split-K over 4 splits, permuted
    (0, 12, 11, 11, 4),       # 256 pair tiles (no split), 64 stages: one tile per pair, TMA-store epilogue
    (0, 12, 11, 14, None),    # K = 16384: two K-chunk launches of 8192, C += by TMA reduce-add
]


@pytest.mark.parametrize("case", range(len(TC_CASES)))
def test_pair_tensor_core_path(case):
    nb, m, n, k, ps = TC_CASES[case]
    ia, ib, ic, dims = _gemm_case(nb, m, n, k, ps)
    got, ref, bound = _run_pair(ia, ib, ic, dims, tb.TN_C64, tb.TN_PATH_TC, seed=10 + case)
    err = np.abs(got - ref)
    ratio = float((err / (tc_tol(2 ** k) * bound + 1e-30)).max())
    _record("tc_err_over_bound", TC_CASES[case], ratio)
    assert ratio <= 1.0, ratio


@pytest.mark.parametrize("case", [(0, 9, 8, 12), (0, 7, 7, 4), (1, 8, 7, 14)])
def test_pair_tensor_core_coherent_operands(case):
    """All-positive real operands: no cancellation, |C| = sum_k |A||B|, the case where
    the step bound tc_tol (relative to sum |A||B|) is tightest."""
    nb, m, n, k = case
    ia, ib, ic, dims = _gemm_case(nb, m, n, k)

    def pos(shape, seed, dtype):
        g = np.random.default_rng(seed)
        return (g.random(shape) + 0.01).astype(np.complex64)

    got, ref, bound = _run_pair(ia, ib, ic, dims, tb.TN_C64, tb.TN_PATH_TC, seed=7, gen=pos)
    ratio = float((np.abs(got - ref) / (tc_tol(2 ** k) * bound)).max())
    _record("tc_err_over_bound_coherent", case, ratio)
    assert ratio <= 1.0, ratio


def _record(name, case, value):
    """achieved error ratios of the step tests, kept for the evidence (gpurun_out/)"""
    import json
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.path.join("gpurun_out", f"{name}.jsonl"), "a") as f:
        f.write(json.dumps({"case": list(case), "value": value}) + "\n")


# (m, n, k): pair kernel (m >= 8, n >= 7; short K on the persistent pair kernel), single-CTA
TC_STAT_CASES = [(9, 8, 4), (9, 8, 5), (9, 8, 6), (9, 8, 7), (9, 8, 10), (10, 10, 12), (7, 7, 6), (7, 7, 10)]


@pytest.mark.parametrize("case", TC_STAT_CASES)
def test_pair_tensor_core_error_statistics(case):
    """Relative error statistics of the complex64 tensor-core GEMM on dense random operands
    (DESIGN.md "Split precision"): bias = Re sum conj(ref)(got - ref) / sum |ref|^2 and
    rms = |got - ref|_2 / |ref|_2 in units of 2^-24.  The TMEM accumulation rounds toward
    zero; without the promotion's debiasing the bias is -14.6 (T = 48 MMA updates per
    chunk), coherent over the steps of a tree.  Required: |bias| <= 3, rms <= 12."""
    m, n, k = case
    ia, ib, ic, dims = _gemm_case(0, m, n, k)
    got, ref, _ = _run_pair(ia, ib, ic, dims, tb.TN_C64, tb.TN_PATH_TC, seed=100 * k + m)
    err = got - ref
    den = float(np.sum(np.abs(ref) ** 2))
    bias = float(np.sum((np.conj(ref) * err).real) / den) / 2 ** -24
    rms = float(np.sqrt(np.sum(np.abs(err) ** 2) / den)) / 2 ** -24
    _record("tc_error_statistics", case, {"bias": bias, "rms": rms})
    assert abs(bias) <= 3.0 and rms <= 12.0, (bias, rms)


def _wide_range(shape, seed, dtype):
    """complex Gaussian entries times 2^u, u uniform in [-12, 12] per entry, with some
    exact zeros and a few entries scaled by 1e-25: the block-scaled fp16x2 split
    must stay at fp32 level relative to sum_k |A||B| (the
    representation floor is 2^-38 of the 128-element chunk maximum, so the guarantee needs
    the dynamic range inside a chunk to stay well below 2^39; 2^24 here)."""
    g = np.random.default_rng(seed)
    x = _rand(shape, seed, dtype).astype(np.complex128)
    x = x * np.exp2(g.uniform(-12, 12, shape))
    flat = x.reshape(-1)
    idx = g.permutation(flat.size)
    flat[idx[: flat.size // 16]] = 0
    flat[idx[flat.size // 16: flat.size // 16 + 8]] *= 1e-25
    return x.astype(np.complex64 if dtype == tb.TN_C64 else np.complex128)


@pytest.mark.parametrize("case", [(0, 7, 8, 9), (1, 6, 7, 12), (0, 7, 7, 4)])
def test_pair_tensor_core_wide_dynamic_range(case):
    """Block-scaled fp16x2 error model: each element x of a
    128-wide K chunk with maximum mx (over re and im) is represented to
    <= 2^-24 |x| + 2^-38 mx, the dropped x1 y1 is <= 2^-24 |x y|, so
    |C - C_ref| <= tol(K) sum_k |A||B| + 2^-37 sum_k (mA |B| + |A| mB).
    Unpermuted layouts, so the chunks are consecutive runs of 128 along K."""
    nb, m, n, k = case
    ia, ib, ic, dims = _gemm_case(nb, m, n, k)
    got, ref, bound = _run_pair(ia, ib, ic, dims, tb.TN_C64, tb.TN_PATH_TC, seed=40, gen=_wide_range)
    assert np.all(np.isfinite(got))
    B_, M_, N_, K_ = 1 << nb, 1 << m, 1 << n, 1 << k
    A = _wide_range([2] * len(ia), 40, tb.TN_C64).reshape(B_, M_, K_).astype(np.complex128)
    Bm = _wide_range([2] * len(ib), 41, tb.TN_C64).reshape(B_, K_, N_).astype(np.complex128)
    ch = min(128, K_)               # the scale chunk (SCALE_LOG2 = 7)
    cm = lambda X: np.maximum(np.abs(X.real), np.abs(X.imag))
    mA = np.repeat(cm(A).reshape(B_, M_, K_ // ch, ch).max(axis=3), ch, axis=2)           # [b][m][k]
    mB = np.repeat(cm(Bm).reshape(B_, K_ // ch, ch, N_).max(axis=2), ch, axis=1)          # [b][k][n]
    floor = np.matmul(mA, np.abs(Bm)) + np.matmul(np.abs(A), mB)
    err = np.abs(got.reshape(B_, M_, N_) - ref.reshape(B_, M_, N_))
    lim = tc_tol(K_) * bound.reshape(B_, M_, N_) + 2.0 ** -37 * floor + 1e-38
    assert np.all(err <= lim), (err / lim).max()


def _zero_chunks(shape, seed, dtype):
    """Gaussian entries with every other run of 128 consecutive elements (one scale
    chunk) set to zero."""
    x = _rand(shape, seed, dtype).reshape(-1).copy()
    for j in range(0, x.size, 256):
        x[j:j + 128] = 0
    return x.reshape(shape)


def test_pair_tensor_core_zero_chunks():
    ia, ib, ic, dims = _gemm_case(0, 7, 7, 8, None)
    got, ref, bound = _run_pair(ia, ib, ic, dims, tb.TN_C64, tb.TN_PATH_TC, seed=41, gen=_zero_chunks)
    assert np.all(np.abs(got - ref) <= c64_tol(2 ** 8) * bound + 1e-30)


# CUDA-core paths for large non-GEMM-shaped steps (device/skinny.cu)
SKINNY_CASES = [
    (0, 3, 4, 12, None),      # 8 x 16 outputs, K = 4096
    (0, 0, 0, 14, 3),         # full contraction to a scalar (one output), permuted
    (2, 2, 3, 11, 4),         # batch 4, permuted layouts
    (0, 6, 2, 10, 5),         # M = 64 rows, N = 4
    (1, 3, 3, 5, None),       # K = 32: a single partial K tile (v1 kernel: below one v2 stage)
    (0, 4, 3, 16, None),      # the configs[4] (4, 3, 26) K-slab shape at K = 65536 (8 groups of 4 x 4)
    (0, 4, 4, 12, 9),         # M = N = 16: 16 groups -> items on halves of X's rows, permuted
    (3, 1, 2, 10, 1),         # batch 8, one 2 x 4 group: 8 warps share its stage iterations
    (0, 0, 0, 20, None),      # configs[3]'s scalar K = 2^20 step: 16 warps take one group's stages in turn
    (10, 4, 4, 7, 2),         # configs[3]'s batched skinny step (gathered: one CTA per batch)
    (6, 0, 0, 10, 3),         # gathered: 64 scalar dot products, 256 lanes of K per output
    (7, 6, 2, 8, 4),          # gathered: M = 64, N = 4, K staged in 4 chunks
    (8, 3, 3, 6, None),       # gathered: 64 outputs x 4 lanes, 256 batches
    (9, 2, 5, 9, 5),          # gathered: 128 outputs x 2 lanes, K = 512 in chunks, permuted
]
WIDE_CASES = [
    (0, 7, 9, 3, None),       # 128 x 512 outputs, K = 8
    (0, 5, 6, 0, 2),          # K = 1 (outer product), ragged tiles (M = 32 rows, N = 64), permuted
    (3, 4, 8, 2, 6),          # batch 8, permuted
    (0, 10, 4, 4, 7),         # N = 16 < tile width
    (2, 3, 12, 4, 3),         # batch 4, K = 16 (complex64: the FFMA2 variant), permuted
]


@pytest.mark.parametrize("dtype", [tb.TN_C64, tb.TN_C128])
@pytest.mark.parametrize("case", range(len(SKINNY_CASES)))
def test_pair_skinny_path(case, dtype):
    nb, m, n, k, ps = SKINNY_CASES[case]
    ia, ib, ic, dims = _gemm_case(nb, m, n, k, ps)
    got, ref, bound = _run_pair(ia, ib, ic, dims, dtype, tb.TN_PATH_SKINNY, seed=50 + case)
    # complex128: fp64 accumulation; complex64: fp32 blocks of <= 8 terms per lane summed
    # in fp64 -- the fp32-path bound for K = 8
    tol = 1e-12 if dtype == tb.TN_C128 else c64_tol(8)
    assert np.all(np.abs(got - ref) <= tol * bound + 1e-30)


@pytest.mark.parametrize("dtype", [tb.TN_C64, tb.TN_C128])
@pytest.mark.parametrize("case", range(len(WIDE_CASES)))
def test_pair_wide_path(case, dtype):
    nb, m, n, k, ps = WIDE_CASES[case]
    ia, ib, ic, dims = _gemm_case(nb, m, n, k, ps)
    got, ref, bound = _run_pair(ia, ib, ic, dims, dtype, tb.TN_PATH_WIDE, seed=60 + case)
    # complex64 accumulates in fp32 (K <= 16): the fp32-path bound
    tol = 1e-12 if dtype == tb.TN_C128 else c64_tol(2 ** k)
    assert np.all(np.abs(got - ref) <= tol * bound + 1e-30)


def test_pair_skinny_gather_off():
    """TN_SKINNY_GATHER=0 (child process): every skinny case through planar packs + the
    staged (TMA) or v1 split-K kernel + the ordered reduction instead of the gathering
    kernel (one CTA per batch and K range) -- within the bound in both dtypes, and the
    two complex128 results within 1e-12 of each other."""
    import subprocess, sys, textwrap
    cases = list(range(len(SKINNY_CASES)))
    code = textwrap.dedent(f"""
        import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
        import numpy as np, test_gpu as T, paper_2208_01498_b200 as tb
        for case in {cases}:
            nb, m, n, k, ps = T.SKINNY_CASES[case]
            ia, ib, ic, dims = T._gemm_case(nb, m, n, k, ps)
            got, ref, bound = T._run_pair(ia, ib, ic, dims, tb.TN_C64, tb.TN_PATH_SKINNY, seed=50 + case)
            assert np.all(np.abs(got - ref) <= T.c64_tol(8) * bound + 1e-30), case
            got, ref, bound = T._run_pair(ia, ib, ic, dims, tb.TN_C128, tb.TN_PATH_SKINNY, seed=50 + case)
            assert np.all(np.abs(got - ref) <= 1e-12 * bound + 1e-30), case
            np.save(f'/tmp/skinny_nogather_{{case}}.npy', got)
        print('ok')
    """)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                       env=dict(os.environ, TN_SKINNY_GATHER="0"),
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
    for case in cases:
        nb, m, n, k, ps = SKINNY_CASES[case]
        ia, ib, ic, dims = _gemm_case(nb, m, n, k, ps)
        got, ref, bound = _run_pair(ia, ib, ic, dims, tb.TN_C128, tb.TN_PATH_SKINNY, seed=50 + case)
        other = np.load(f'/tmp/skinny_nogather_{case}.npy')
        assert np.all(np.abs(got - other) <= 1e-12 * bound + 1e-30), case


def test_pair_skinny_k_slabs():
    """skinny path with K-slabs (pack cap lowered in a child process): the slab sums
    accumulate into C."""
    import subprocess, sys, textwrap
    code = textwrap.dedent("""
        import sys; sys.path.insert(0, '.')
        sys.path.insert(0, 'tests')
        import numpy as np, test_gpu as T, paper_2208_01498_b200 as tb
        for dt in (tb.TN_C64, tb.TN_C128):
            ia, ib, ic, dims = T._gemm_case(1, 3, 2, 14, 8)
            got, ref, bound = T._run_pair(ia, ib, ic, dims, dt, tb.TN_PATH_SKINNY, seed=33)
            tol = 1e-12 if dt == tb.TN_C128 else T.c64_tol(8)
            assert np.all(np.abs(got - ref) <= tol * bound + 1e-30), (np.abs(got - ref) / bound).max()
        print('ok')
    """)
    env = dict(os.environ, TN_PACK_CAP_LOG2="12")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


DMMA_CASES = [
    (0, 6, 6, 4, None),       # one 64x64 tile, K = 16
    (0, 5, 7, 3, 2),          # ragged M = 32, N = 128, K = 8, permuted
    (2, 7, 6, 9, 4),          # batch 4, K = 512 (32 stages), permuted (tail split: 8 tiles, K in 4)
    (0, 9, 9, 6, None),       # 64 tiles, K too short to split
    (6, 10, 6, 9, 5),         # configs[3]'s dominant step: 1024 tiles = 3 waves + 136 (tail split: K in 2)
    (0, 9, 9, 10, None),      # 64 tiles, K = 1024 (tail split: one launch of clusters of 4)
    (0, 5, 7, 8, 2),          # ragged M = 32, 2 tiles (tail split: K in 2)
    (2, 9, 8, 8, 3),          # 128 tiles, K = 256, batch 4, permuted (tail split: K in 2)
]


@pytest.mark.parametrize("case", range(len(DMMA_CASES)))
def test_pair_complex128_dmma_path(case):
    nb, m, n, k, ps = DMMA_CASES[case]
    ia, ib, ic, dims = _gemm_case(nb, m, n, k, ps)
    got, ref, bound = _run_pair(ia, ib, ic, dims, tb.TN_C128, tb.TN_PATH_TC, seed=20 + case)
    assert np.all(np.abs(got - ref) <= 1e-13 * bound + 1e-300)


def test_pair_complex128_dmma_tail_split():
    """TN_DMMA_TAIL=1 (child process): the partial last wave of tiles runs as a second
    launch with K split over clusters of 2 or 4 CTAs, the leader adding the partial
    accumulators over DSMEM in rank order -- within the DMMA bound, bit-identical over two
    runs, and within 1e-13 Σ|A||B| of the one-launch default (only the order of the K
    summation differs)."""
    import subprocess, sys, textwrap
    code = textwrap.dedent("""
        import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
        import numpy as np, test_gpu as T, paper_2208_01498_b200 as tb
        for case in (2, 4, 5, 6, 7):
            nb, m, n, k, ps = T.DMMA_CASES[case]
            ia, ib, ic, dims = T._gemm_case(nb, m, n, k, ps)
            got, ref, bound = T._run_pair(ia, ib, ic, dims, tb.TN_C128, tb.TN_PATH_TC, seed=20 + case)
            assert np.all(np.abs(got - ref) <= 1e-13 * bound + 1e-300), case
            again, _, _ = T._run_pair(ia, ib, ic, dims, tb.TN_C128, tb.TN_PATH_TC, seed=20 + case)
            assert np.array_equal(got, again), case
            np.save(f'/tmp/dmma_tail_{case}.npy', got)
        print('ok')
    """)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                       env=dict(os.environ, TN_DMMA_TAIL="1"),
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
    for case in (2, 4, 5, 6, 7):
        nb, m, n, k, ps = DMMA_CASES[case]
        ia, ib, ic, dims = _gemm_case(nb, m, n, k, ps)
        got, ref, bound = _run_pair(ia, ib, ic, dims, tb.TN_C128, tb.TN_PATH_TC, seed=20 + case)
        split = np.load(f'/tmp/dmma_tail_{case}.npy')
        assert np.all(np.abs(got - split) <= 1e-13 * bound + 1e-300), case


def test_pair_tensor_core_k_slabs(monkeypatch):
    """K-slab packing (bounded pack buffers): forced by lowering the pack cap in child
    processes (the cap is read once per process).  Cap 2^13: K-slabs and row slabs of
    single-CTA and pair steps, incl. (0, 9, 8, 10): 32 K-slabs on the persistent pair
    kernel, C += by TMA reduce-add; cap 2^23: (0, 12, 11, 14), 8 K-slabs of 64 stages on
    the one-tile-per-pair kernel, 512 CTAs (no split-K), reduce-add from its epilogue;
    with a batch index and permuted layouts: cap 2^21 (1, 11, 10, 12) on the persistent
    kernel, cap 2^24 (1, 12, 11, 13) on the one-tile-per-pair kernel."""
    import subprocess, sys, textwrap
    code = textwrap.dedent("""
        import sys; sys.path.insert(0, '.')
        sys.path.insert(0, 'tests')
        import numpy as np, test_gpu as T, paper_2208_01498_b200 as tb
        for case in CASES:
            nb, m, n, k, ps = case
            ia, ib, ic, dims = T._gemm_case(nb, m, n, k, ps)
            got, ref, bound = T._run_pair(ia, ib, ic, dims, tb.TN_C64, tb.TN_PATH_TC, seed=31)
            err = np.abs(got - ref)
            assert np.all(err <= T.c64_tol(2 ** k) * bound + 1e-30), (case, (err / bound).max())
        print('ok')
    """)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for cap, cases in (("13", [(0, 7, 7, 9, 1), (1, 6, 7, 14, 2), (0, 10, 7, 4, None), (1, 10, 7, 4, 3),
                               (0, 11, 8, 4, 5), (0, 9, 8, 10, None)]),
                       ("21", [(1, 11, 10, 12, 6)]),
                       ("23", [(0, 12, 11, 14, None)]),
                       ("24", [(1, 12, 11, 13, 2)])):
        env = dict(os.environ, TN_PACK_CAP_LOG2=cap)
        r = subprocess.run([sys.executable, "-c", code.replace("CASES", repr(cases))], capture_output=True,
                           text=True, env=env, cwd=root)
        assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_plan_with_bounded_pack_buffers():
    """A whole plan (6x6 lattice, tensor-core steps) with the pack cap lowered to 2^12 so
    its GEMM steps run in K-slabs or row slabs; amplitudes against the oracle (child
    process: the cap is read once per process)."""
    import subprocess, sys, textwrap
    code = textwrap.dedent("""
        import sys; sys.path.insert(0, '.')
        sys.path.insert(0, 'tests')
        import test_gpu as T, paper_2208_01498_b200 as tb
        from tn_inputs import lattice_cz
        plan = T._plan_vs_oracle(lattice_cz(6, 6, 12, 8), tb.TN_C64, seed=0, n_bits=2)
        st = plan.steps()
        assert (st[:, 0] == tb.TN_PATH_TC).sum() >= 1
        print('ok')
    """)
    env = dict(os.environ, TN_PACK_CAP_LOG2="12")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_pair_tc_matches_small_path():
    ia, ib, ic, dims = _gemm_case(1, 7, 7, 6, 9)
    g1, ref, bound = _run_pair(ia, ib, ic, dims, tb.TN_C64, tb.TN_PATH_TC, seed=3)
    g2, _, _ = _run_pair(ia, ib, ic, dims, tb.TN_C64, tb.TN_PATH_SMALL, seed=3)
    assert np.all(np.abs(g1 - g2) <= 2 * c64_tol(2 ** 6) * bound + 1e-30)


# ------------------------------------------------------------------ plans ----
def _amp_tol(dtype, n):
    return (1e-10 if dtype == tb.TN_C128 else 1e-5), 2.0 ** (-n / 2)


def _plan_vs_oracle(circ, dtype, seed, hyper=False, max_log2_size=0, n_bits=4, with_zero=True):
    _cuda()
    on = build_network(circ, diag_hyper=hyper)
    osteps, _ = find_order(on, seed=seed, max_log2_size=max_log2_size)
    cn = tb.Network.from_circuit(circ, diag_hyper=hyper)
    co = tb.Order(cn, seed=seed, max_log2_size=max_log2_size)
    assert co.steps() == osteps                       # bit-identical order
    plan = tb.Plan(cn, co, dtype=dtype)
    bits = random_bitstrings(circ.n, n_bits, seed)
    if with_zero:
        bits = np.vstack([np.zeros((1, circ.n), np.uint8), bits])
    got = plan.amplitudes(bits)
    tol, scale = _amp_tol(dtype, circ.n)
    for x, g in zip(bits, got):
        want = contract_tree(on, osteps, x)
        assert abs(g - want) <= tol * max(abs(want), scale), (x, g, want)
    return plan


def test_config0_complex128_all_bitstrings():
    """configs[0]: 4x4 depth 8, complex128, <0|C|0> + 16 seeded bitstrings."""
    _plan_vs_oracle(config_circuit(0), tb.TN_C128, seed=0, n_bits=16)


def test_config0_complex64():
    _plan_vs_oracle(config_circuit(0), tb.TN_C64, seed=0, n_bits=16)


def test_plan_with_slicing_matches_unsliced_oracle():
    c = lattice_cz(5, 5, 8, 4)
    plan = _plan_vs_oracle(c, tb.TN_C128, seed=1, max_log2_size=12, n_bits=3)
    assert plan.info()["n_slices"] > 1


def test_plan_slices_partition_the_amplitude():
    c = lattice_cz(4, 5, 8, 6)
    cn = tb.Network.from_circuit(c)
    co = tb.Order(cn, seed=2, max_log2_size=10)
    plan = tb.Plan(cn, co, dtype=tb.TN_C128)
    ns = plan.info()["n_slices"]
    x = random_bitstrings(c.n, 1, 5)[0]
    full = plan.contract(x)
    parts = sum(plan.contract(x, s, s + 1) for s in range(ns))
    assert abs(full - parts) < 1e-12


def test_iqp_hyperedges_complex128():
    _plan_vs_oracle(iqp(5, 2, 7), tb.TN_C128, seed=3, hyper=True, n_bits=6)


def test_sycamore_small_complex64():
    _plan_vs_oracle(sycamore(4, 3), tb.TN_C64, seed=4, n_bits=2, max_log2_size=22)


def test_plan_uses_tensor_cores_and_matches_oracle():
    """6x6 depth 12: several GEMM-shaped steps go to tcgen05 inside one plan."""
    c = lattice_cz(6, 6, 12, 8)
    plan = _plan_vs_oracle(c, tb.TN_C64, seed=5, n_bits=2, with_zero=False)
    assert plan.info()["n_steps_tc"] >= 1


def test_c_then_cdagger_identity_on_gpu():
    c = lattice_cz(5, 5, 6, 9)
    cc = concat(c, inverse_circuit(c))
    cn = tb.Network.from_circuit(cc)
    co = tb.Order(cn, seed=0, max_log2_size=24)
    plan = tb.Plan(cn, co, dtype=tb.TN_C64)
    assert abs(plan.contract(np.zeros(c.n, np.uint8)) - 1.0) < 1e-5


def test_contract_device_accumulates_on_device():
    dev = _cuda()
    c = config_circuit(0)
    cn = tb.Network.from_circuit(c)
    co = tb.Order(cn, seed=0)
    plan = tb.Plan(cn, co, dtype=tb.TN_C128)
    x = random_bitstrings(c.n, 1, 1)[0]
    bits = torch.from_numpy(x).to(dev)
    amp = torch.zeros(1, dtype=torch.complex128, device=dev)
    plan.contract_device(bits.data_ptr(), 0, 1, amp.data_ptr(), torch.cuda.current_stream().cuda_stream)
    plan.contract_device(bits.data_ptr(), 0, 1, amp.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert abs(amp.item() - 2 * plan.contract(x)) < 1e-13


@pytest.mark.slow
def test_config3_full_size_sampled_amplitudes():
    """configs[3] (IQP 10x10, r = 2, complex128, hyperedges): plan at full size; two of
    the 256 seeded amplitudes against the oracle along its (bit-identical) order."""
    c = config_circuit(3)
    plan = _plan_vs_oracle(c, tb.TN_C128, seed=0, hyper=True, n_bits=1, with_zero=False)
    assert plan.info()["n_steps_tc"] >= 1
    # the plan's steps went through the gathered DMMA, wide and gathered skinny kernels
    paths = set(int(p) for p in plan.steps()[:, 0])
    assert {tb.TN_PATH_TC, tb.TN_PATH_WIDE, tb.TN_PATH_SKINNY, tb.TN_PATH_SMALL} <= paths, paths


# ------------------------------------------------ full-size config 1 ------
def test_config1_full_size_biggest_gemm_sampled():
    """configs[1] (8x8 depth 16, complex64): the bench's plan (best of 256 hierarchies,
    bench.SPEC's slicing target); take its largest tensor-core step whose operands
    and result all fit in 2^31 entries (the bench plan's biggest steps hold 2^32-entry
    operands that cannot be materialised again beside it) and run that GEMM shape through
    tn_contract_pair -- the same kernels, tiles, slabs and grid as in the plan -- on random
    operands; 64 sampled outputs against complex128 dot products."""
    dev = _cuda()
    c = config_circuit(1)
    cn = tb.Network.from_circuit(c)
    plan = None
    import bench
    tgt = bench.SPEC[1]["slice_log"]
    co = tb.Order(cn, seed=0, n_seeds=256, max_log2_size=tgt)
    plan = tb.Plan(cn, co, dtype=tb.TN_C64)
    st = plan.steps()
    tc = st[st[:, 0] == tb.TN_PATH_TC]
    fits = [r for r in tc if max(r[1] + r[2] + r[4], r[1] + r[3] + r[4], r[1] + r[2] + r[3]) <= 31]
    assert len(fits) > 0
    big = max(fits, key=lambda r: int(r[1] + r[2] + r[3] + r[4]))
    nb, m, n, k = (int(v) for v in big[1:5])
    del plan
    torch.cuda.empty_cache()
    B_, M_, N_, K_ = 1 << nb, 1 << m, 1 << n, 1 << k
    g = torch.Generator(device=dev).manual_seed(1)
    A = torch.randn(B_, M_, K_, dtype=torch.complex64, device=dev, generator=g)
    Bm = torch.randn(B_, K_, N_, dtype=torch.complex64, device=dev, generator=g)
    Cm = torch.empty(B_, M_, N_, dtype=torch.complex64, device=dev)
    ids = list(range(nb + m + n + k))
    bt, mm, nn, kk = ids[:nb], ids[nb:nb + m], ids[nb + m:nb + m + n], ids[nb + m + n:]
    tb.contract_pair(tb.TN_C64, A.data_ptr(), bt + mm + kk, Bm.data_ptr(), bt + kk + nn, Cm.data_ptr(),
                     bt + mm + nn, [2] * len(ids), tb.TN_PATH_TC)
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    for _ in range(64):
        b, i, j = int(rng.integers(B_)), int(rng.integers(M_)), int(rng.integers(N_))
        a_row = A[b, i, :].cpu().numpy().astype(np.complex128)
        b_col = Bm[b, :, j].cpu().numpy().astype(np.complex128)
        want = np.dot(a_row, b_col)
        bound = np.dot(np.abs(a_row), np.abs(b_col))
        assert abs(Cm[b, i, j].item() - want) <= c64_tol(K_) * bound


# ------------------------------------------- full-size sliced networks ------
@pytest.mark.parametrize("ci,tgt", [(1, 22), (2, 22), (4, 22)])
def test_full_size_config_slices(ci, tgt):
    """configs[1], [2] (Sycamore-53 m=14) and [4] ((2+1)D 12x12 depth 20) at full size in
    complex64, sliced until every tensor has <= 2^tgt entries (slice
    bits: 52, 68, 163): order and sliced indices bit-identical to the oracle's, and
    three sliced sub-contractions of one bitstring against oracle.contract_slice.
    Slice ids are int64, so with > 63 sliced bits the higher sliced indices stay 0.
    Slices of config 4 reach 2^-165 unscaled, below complex64: this also pins the
    plan's leaf scaling.  Tolerance: 1e-5 relative to
    max(|ref|, 2^(-n/2) / 2^(slice_bits/2)), the RMS of one slice of an amplitude."""
    _cuda()
    c = config_circuit(ci)
    on = build_network(c)
    osteps, _ = find_order(on, seed=0, max_log2_size=tgt)
    sl = choose_slices(on, osteps, tgt)
    cn = tb.Network.from_circuit(c)
    co = tb.Order(cn, seed=0, max_log2_size=tgt)
    assert co.steps() == osteps
    assert co.slices() == sl
    plan = tb.Plan(cn, co, dtype=tb.TN_C64)
    info = plan.info()
    nbits = info["slice_bits"]
    assert nbits == sum(on.log2dim(i) for i in sl)
    x = random_bitstrings(c.n, 1, 11)[0]
    rng = np.random.default_rng(ci)
    top = min(nbits, 62)
    for sid in [0, int(rng.integers(1 << top)), int(rng.integers(1 << top))]:
        fixed, shift = {}, 0
        for i in reversed(sl):                      # last sliced index fastest
            fixed[i] = (sid >> shift) & (on.dims[i] - 1) if shift < 63 else 0
            shift += on.log2dim(i)
        want = contract_slice(on, osteps, x, fixed)
        got = plan.contract(x, sid, sid + 1)
        scale = 2.0 ** (-c.n / 2 - nbits / 2)
        assert abs(got - want) <= 1e-5 * max(abs(want), scale), (sid, got, want)


def test_config1_slices_with_bounded_pack_buffers():
    """configs[1] at full size, slicing target 2^22, with the pack cap lowered to 2^18 so
    its large steps run in K-slabs / row slabs (as the bench's 2^34 plan does at the
    default cap): slices against oracle.contract_slice (child process: the cap is read
    once per process)."""
    import subprocess, sys, textwrap
    code = textwrap.dedent("""
        import sys; sys.path.insert(0, '.')
        sys.path.insert(0, 'tests')
        import test_gpu as T
        T.test_full_size_config_slices(1, 22)
        print('ok')
    """)
    env = dict(os.environ, TN_PACK_CAP_LOG2="18")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_lanes_with_sliced_plan():
    """Lanes on a sliced plan: every lane walks all slices of its bitstrings (slice
    counter and fp64 accumulator per lane) -- same amplitudes as one lane, and as the
    unsliced oracle."""
    _cuda()
    c = lattice_cz(5, 5, 8, 4)
    on = build_network(c)
    osteps, _ = find_order(on, seed=1, max_log2_size=12)
    cn = tb.Network.from_circuit(c)
    co = tb.Order(cn, seed=1, max_log2_size=12)
    assert co.steps() == osteps
    plan = tb.Plan(cn, co, dtype=tb.TN_C128)
    assert plan.info()["n_slices"] > 1
    bits = random_bitstrings(c.n, 5, 8)
    single = plan.amplitudes(bits)
    plan.set_lanes(2)
    multi = plan.amplitudes(bits)
    assert np.array_equal(single, multi)
    for x, g in zip(bits, multi):
        want = contract_tree(on, osteps, x)
        assert abs(g - want) <= 1e-10 * max(abs(want), 2.0 ** (-c.n / 2))


def test_lanes_concurrent_amplitudes():
    """tn_plan_set_lanes: configs[0] (complex128) and a 6x6 complex64 lattice with
    tensor-core steps, 3 lanes, amplitudes of 7 bitstrings against the oracle (lane j mod 3
    contracts bitstring j concurrently) and bit-identical to the single-lane plan."""
    _cuda()
    for circ, dtype in ((config_circuit(0), tb.TN_C128), (lattice_cz(6, 6, 12, 8), tb.TN_C64)):
        on = build_network(circ)
        osteps, _ = find_order(on, seed=0)
        cn = tb.Network.from_circuit(circ)
        co = tb.Order(cn, seed=0)
        p1 = tb.Plan(cn, co, dtype=dtype)
        bits = random_bitstrings(circ.n, 7, 5)
        single = p1.amplitudes(bits)
        p1.set_lanes(3)
        multi = p1.amplitudes(bits)
        assert np.array_equal(single, multi)
        tol, scale = _amp_tol(dtype, circ.n)
        for x, g in zip(bits, multi):
            want = contract_tree(on, osteps, x)
            assert abs(g - want) <= tol * max(abs(want), scale)


def test_amplitudes_empty_batch_and_fewer_bitstrings_than_lanes():
    """Edge cases of tn_amplitudes (include/tn.h): an empty batch returns no amplitudes
    and leaves the plan usable; with more lanes than bitstrings (2 and 1 bitstrings on 4
    lanes: idle lanes, and the n_bits < 2 single-lane route) the amplitudes are
    bit-identical to the single-lane plan's and match the oracle."""
    _cuda()
    c = lattice_cz(5, 5, 8, 4)
    on = build_network(c)
    osteps, _ = find_order(on, seed=1, max_log2_size=12)
    cn = tb.Network.from_circuit(c)
    co = tb.Order(cn, seed=1, max_log2_size=12)
    assert co.steps() == osteps
    for lanes in (1, 4):
        plan = tb.Plan(cn, co, dtype=tb.TN_C128)
        bits = random_bitstrings(c.n, 2, 11)
        single = plan.amplitudes(bits)
        if lanes > 1:
            plan.set_lanes(lanes)
        empty = plan.amplitudes(np.zeros((0, c.n), np.uint8))
        assert empty.shape == (0,) and empty.dtype == np.complex128
        assert np.array_equal(plan.amplitudes(bits), single)
        assert np.array_equal(plan.amplitudes(bits[:1]), single[:1])
        for x, g in zip(bits, single):
            want = contract_tree(on, osteps, x)
            assert abs(g - want) <= 1e-10 * max(abs(want), 2.0 ** (-c.n / 2))


def test_bench_plan_slice_self_consistent():
    """The bench's own plan (configs[1], best of 256 hierarchies, bench.SPEC's slicing
    target, 2^30-entry pack cap: K-slabs, row slabs, CTA pairs, persistent tiles) is
    beyond the oracle; run one of its slices three ways -- default, pack cap 2^28 (other
    slab structure), single-CTA GEMM (no cta_group::2 / persistent kernels) -- and require
    agreement to 1e-5 of the RMS slice (child processes: plans of ~180 GB each)."""
    import subprocess, sys, textwrap
    code = textwrap.dedent("""
        import sys; sys.path.insert(0, '.')
        import numpy as np, paper_2208_01498_b200 as tb
        from tn_inputs import config_circuit, random_bitstrings
        c = config_circuit(1)
        net = tb.Network.from_circuit(c)
        import bench
        tgt = bench.SPEC[1]["slice_log"]
        o = tb.Order(net, seed=0, n_seeds=256, max_log2_size=tgt)
        p = tb.Plan(net, o, dtype=tb.TN_C64)
        x = random_bitstrings(c.n, 1, 1)[0]
        ids = p.contributing_slice_ids(x, 0, 4)
        a = p.contract(x, 0, ids[-1] + 1)   # the first 4 contributing slices (zero ones skipped)
        print(repr((tgt, p.info()["slice_bits"], a.real, a.imag)))
    """)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for env in ({}, {"TN_PACK_CAP_LOG2": "28"}, {"TN_GEMM_PAIR": "0", "TN_GEMM_PERSIST": "0"}):
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                           env=dict(os.environ, **env), cwd=root, timeout=900)
        assert r.returncode == 0, r.stdout + r.stderr
        res.append(eval(r.stdout.strip().splitlines()[-1]))
    tgt, bits = res[0][0], res[0][1]
    assert all(r[0] == tgt and r[1] == bits for r in res)
    vals = [complex(r[2], r[3]) for r in res]
    scale = 2.0 ** (-64 / 2 - bits / 2)
    assert max(abs(v) for v in vals) > 0
    for v in vals[1:]:
        assert abs(v - vals[0]) <= 1e-5 * max(abs(vals[0]), scale), vals


def test_zero_slices_skipped():
    """Provably zero slices (a leaf whose only sliced index is fixed against its bound
    output legs vanishes): tn_contributing_slices counts fewer slices than the plan has,
    and tn_contract (host bitstring, skipping them) equals the device-bitstring sum over
    all slices and the unsliced oracle."""
    dev = _cuda()
    found = False
    for cseed, seed, tgt in ((30, 2, 3), (31, 2, 3)):      # slicing a CZ bond next to an output leg
        c = lattice_cz(3, 4, 4, cseed)
        on = build_network(c)
        osteps, _ = find_order(on, seed=seed, max_log2_size=tgt)
        cn = tb.Network.from_circuit(c)
        co = tb.Order(cn, seed=seed, max_log2_size=tgt)
        assert co.steps() == osteps
        plan = tb.Plan(cn, co, dtype=tb.TN_C128)
        ns = plan.info()["n_slices"]
        for x in random_bitstrings(c.n, 6, seed):
            k = plan.contributing_slices(x)
            assert 1 <= k <= ns
            if k == ns:
                continue
            found = True
            got = plan.contract(x)
            bits = torch.from_numpy(x).to(dev)
            amp = torch.zeros(1, dtype=torch.complex128, device=dev)
            plan.contract_device(bits.data_ptr(), 0, ns, amp.data_ptr(), torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            want = contract_tree(on, osteps, x)
            assert abs(got - amp.item()) <= 1e-12 * max(abs(want), 2.0 ** (-c.n / 2))
            assert abs(got - want) <= 1e-10 * max(abs(want), 2.0 ** (-c.n / 2))
    assert found, "no plan with provably zero slices in the sample"


def test_degenerate_circuits_on_gpu():
    """Degenerate circuits (one qubit, product state, no gates, disconnected components;
    tests/degenerate.py) in both dtypes: every amplitude against its closed form and
    the oracle, and an empty slice range contributes exactly 0."""
    _cuda()
    from degenerate import degenerate_circuits, all_bitstrings
    for c, amp in degenerate_circuits():
        on = build_network(c)
        osteps, _ = find_order(on, seed=0)
        cn = tb.Network.from_circuit(c)
        co = tb.Order(cn, seed=0)
        assert co.steps() == osteps
        xs = all_bitstrings(c.n)
        for dtype in (tb.TN_C128, tb.TN_C64):
            plan = tb.Plan(cn, co, dtype=dtype)
            got = plan.amplitudes(xs)
            tol = 1e-12 if dtype == tb.TN_C128 else 1e-6
            for x, g in zip(xs, got):
                assert abs(g - amp(x)) <= tol, (c.name, dtype, x, g, amp(x))
                assert abs(g - contract_tree(on, osteps, x)) <= tol
                assert plan.contract(x, 0, 0) == 0


def test_pair_misaligned_output_is_an_error_not_a_crash():
    """tn.h: C must be 16-byte aligned on the tensor-core pair path (TMA stores).  A C
    view 8 bytes off is refused with an error (TN_ECUDA from the tensor-map encode), the
    library stays usable, and the next aligned call is correct."""
    dev = _cuda()
    nb, m, n, k = 0, 8, 7, 6
    ia, ib, ic, dims = _gemm_case(nb, m, n, k)
    A = torch.randn(1 << (m + k), dtype=torch.complex64, device=dev)
    B = torch.randn(1 << (n + k), dtype=torch.complex64, device=dev)
    Cbuf = torch.zeros((1 << (m + n)) + 1, dtype=torch.complex64, device=dev)
    with pytest.raises(tb.TnError):
        tb.contract_pair(tb.TN_C64, A.data_ptr(), ia, B.data_ptr(), ib, Cbuf[1:].data_ptr(), ic, dims, tb.TN_PATH_TC)
    torch.cuda.synchronize()
    got, ref, bound = _run_pair(ia, ib, ic, dims, tb.TN_C64, tb.TN_PATH_TC, seed=3)
    assert np.all(np.abs(got - ref) <= tc_tol(2 ** k) * bound + 1e-30)


@pytest.mark.parametrize("dtype", [tb.TN_C64, tb.TN_C128])
def test_pair_degenerate_pack_shapes(dtype):
    """Operands with fewer than 8 entries per batch (rows + K bits < 3) cannot be packed
    (the pack kernels write 8 consecutive elements per thread): AUTO sends such steps to
    the small path and is exact; forcing a packed path is refused with an error and
    leaves C untouched (m = 0 / n = 0 with batch bits)."""
    dev = _cuda()
    for nb, m, n, k in ((16, 0, 2, 1), (5, 0, 2, 1), (17, 2, 0, 1), (4, 0, 3, 1)):
        ia, ib, ic, dims = _gemm_case(nb, m, n, k)
        got, ref, bound = _run_pair(ia, ib, ic, dims, dtype, tb.TN_PATH_AUTO, seed=nb + m)
        tol = 1e-12 if dtype == tb.TN_C128 else c64_tol(2 ** k)
        assert np.all(np.abs(got - ref) <= tol * bound + 1e-30), (nb, m, n, k)
    tdt = torch.complex64 if dtype == tb.TN_C64 else torch.complex128
    for (nb, m, n, k), path in (((16, 0, 2, 1), tb.TN_PATH_WIDE), ((4, 0, 3, 1), tb.TN_PATH_SKINNY),
                                ((4, 0, 6, 2), tb.TN_PATH_TC)):
        ia, ib, ic, dims = _gemm_case(nb, m, n, k)
        A = torch.ones(1 << (nb + m + k), dtype=tdt, device=dev)
        B = torch.ones(1 << (nb + n + k), dtype=tdt, device=dev)
        Cbuf = torch.full((2 << (nb + m + n),), 7.0, dtype=tdt, device=dev)
        with pytest.raises(tb.TnError):
            tb.contract_pair(dtype, A.data_ptr(), ia, B.data_ptr(), ib, Cbuf.data_ptr(), ic, dims, path)
        torch.cuda.synchronize()
        assert bool((Cbuf == 7.0).all()), (nb, m, n, k, path)


def test_plans_on_two_devices_when_present():
    """The >48 KB shared-memory attribute is per device: plans created on every
    visible device run their tensor-core steps and agree with the oracle."""
    _cuda()
    c = lattice_cz(6, 6, 12, 8)
    on = build_network(c)
    osteps, _ = find_order(on, seed=0)
    cn = tb.Network.from_circuit(c)
    co = tb.Order(cn, seed=0)
    x = random_bitstrings(c.n, 1, 5)[0]
    want = contract_tree(on, osteps, x)
    for dev in range(min(torch.cuda.device_count(), 2)):
        plan = tb.Plan(cn, co, dtype=tb.TN_C64, device=dev)
        assert plan.info()["n_steps_tc"] > 0
        got = plan.amplitudes(np.array([x]))[0]
        assert abs(got - want) <= 1e-5 * max(abs(want), 2.0 ** (-c.n / 2))


GUARD_CASES = [
    (tb.TN_PATH_SKINNY, 9, 2, 5, 9, 5),     # gathered skinny, chunked K
    (tb.TN_PATH_SKINNY, 0, 0, 0, 14, 3),    # gathered skinny, K ranges + ordered reduction
    (tb.TN_PATH_SKINNY, 1, 3, 2, 14, 8),    # gathered skinny, 2 batches x K ranges, permuted
    (tb.TN_PATH_WIDE, 2, 5, 6, 2, 4),       # wide, one CTA per tile
    (tb.TN_PATH_TC, 3, 9, 7, 8, 2),         # DMMA (complex128) / tcgen05 (complex64)
    (tb.TN_PATH_SMALL, 2, 3, 3, 4, 1),      # small wave
]


@pytest.mark.parametrize("dtype", [tb.TN_C64, tb.TN_C128])
@pytest.mark.parametrize("case", range(len(GUARD_CASES)))
def test_pair_writes_stay_in_bounds(case, dtype):
    """C is written exactly where it lives: the output sits between two guard bands of
    4096 sentinel entries in one allocation; after the step every sentinel is intact and
    every output element finite and within its bound of the oracle."""
    dev = _cuda()
    path, nb, m, n, k, ps = GUARD_CASES[case]
    ia, ib, ic, dims = _gemm_case(nb, m, n, k, ps)
    A = _rand([dims[i] for i in ia], 70 + case, dtype)
    B = _rand([dims[i] for i in ib], 71 + case, dtype)
    tdt = torch.complex64 if dtype == tb.TN_C64 else torch.complex128
    sc = [dims[i] for i in ic]
    n_c = int(np.prod(sc)) if sc else 1
    G = 4096
    buf = torch.full((n_c + 2 * G,), complex(1234.5, -6789.25), dtype=tdt, device=dev)
    tA, tB = torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev)
    torch.cuda.synchronize()
    tb.contract_pair(dtype, tA.data_ptr(), ia, tB.data_ptr(), ib, buf[G:].data_ptr(), ic, dims, path)
    torch.cuda.synchronize()
    h = buf.cpu().numpy()
    assert np.all(h[:G] == complex(1234.5, -6789.25)) and np.all(h[G + n_c:] == complex(1234.5, -6789.25))
    got = h[G:G + n_c].reshape(sc) if sc else h[G:G + 1].reshape(())
    ref_inds, ref = oracle_pair(list(ia), A.astype(np.complex128), list(ib), B.astype(np.complex128), ic, dims)
    _, bound = oracle_pair(list(ia), np.abs(A).astype(np.complex128), list(ib), np.abs(B).astype(np.complex128), ic, dims)
    perm = [ref_inds.index(i) for i in ic]
    ref = np.transpose(ref, perm) if perm else ref
    bound = np.abs(np.transpose(bound, perm) if perm else bound)
    tol = (1e-12 if dtype == tb.TN_C128 else (tc_tol(1 << k) if path == tb.TN_PATH_TC else c64_tol(1 << min(k, 3))))
    assert np.all(np.isfinite(got))
    assert np.all(np.abs(got - ref) <= tol * bound + 1e-30)
