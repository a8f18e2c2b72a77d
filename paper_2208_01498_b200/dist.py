"""Multi-GPU partitioning of the contraction (one process per GPU, torch.distributed).

Two ways the path shards (BASELINE north_star "Index slicing and multi-GPU
partitioning"); both are used by bench.py and by the tests, so the code that would run
on 8 GPUs is the code the tests run:
  * bitstrings: independent amplitudes -> contiguous blocks of the batch per rank, no
    data-path collective;
  * slices: the sliced sub-contractions of ONE amplitude ("index
    slicing") are independent -> disjoint contiguous blocks of its (contributing)
    slices per rank, the partial amplitudes summed with ONE all-reduce (NCCL over
    NVLink on the GPU path, gloo in the CPU tests).
Every function takes the world size / rank explicitly or from the default process
group; nothing here does contraction arithmetic.  shared_order: the host order search
runs once per job (rank 0) and is broadcast.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def world_rank(group=None):
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def block_range(n: int, world: int, rank: int):
    """Contiguous, balanced block [lo, hi) of n items for `rank` (blocks of all ranks are
    disjoint and cover [0, n); sizes differ by at most one)."""
    q, r = divmod(n, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def slice_block(live_slices, world: int, rank: int):
    """This rank's block of the slices of one amplitude: `live_slices` is the list of
    slice ids to contract (the contributing ones, tn_contributing_slice_ids), the ranks
    get disjoint contiguous blocks, so the all-reduced sum counts every slice once."""
    lo, hi = block_range(len(live_slices), world, rank)
    return list(live_slices[lo:hi])


def bitstring_steps(contributing_ids, rows, count: int):
    """Work items (row, slice) for `count` steps over this rank's bitstrings `rows`
    (indices into the batch), one contributing slice per step, bitstring by bitstring:
    contributing_ids(row, n) -> the first n contributing slice ids of that bitstring.
    No (row, slice) pair repeats; fewer than `count` items if the rows run out."""
    items = []
    for r in rows:
        if len(items) >= count:
            break
        for s in contributing_ids(r, count - len(items)):
            items.append((r, s))
    return items


def shared_order(find_order, import_order, device=None):
    """One host order search per job: rank 0 runs find_order() (tn_find_order, with all
    the host's cores), its steps, sliced indices and median-fallback count go to every
    rank by two broadcasts of the default group, and the other ranks build the same
    order with import_order(steps, slices, median_fallbacks) (tn_order_import).  Every
    rank then holds the identical tree by construction (find_order is deterministic
    anyway; this saves N - 1 searches that would share the host's cores).  find_order()
    returns an object with steps(), slices() and info()["median_fallbacks"]."""
    world, rank = world_rank()
    if world == 1:
        return find_order()
    o = find_order() if rank == 0 else None
    hdr = torch.zeros(3, dtype=torch.int64, device=device)
    if rank == 0:
        steps, slices = o.steps(), o.slices()
        hdr[0], hdr[1], hdr[2] = len(steps), len(slices), int(o.info()["median_fallbacks"])
    dist.broadcast(hdr, src=0)
    n_st, n_sl, mf = (int(v) for v in hdr.cpu().tolist())
    body = torch.zeros(max(2 * n_st + n_sl, 1), dtype=torch.int64, device=device)
    if rank == 0:
        flat = [v for ab in steps for v in ab] + list(slices)
        if flat:
            body[:len(flat)] = torch.tensor(flat, dtype=torch.int64)
    dist.broadcast(body, src=0)
    if rank == 0:
        return o
    v = body.cpu().tolist()
    return import_order([(v[2 * k], v[2 * k + 1]) for k in range(n_st)], v[2 * n_st:2 * n_st + n_sl], mf)


def allreduce_sum_(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place SUM over ranks (the one data-path collective of the sliced path);
    a no-op without a process group / at world size 1."""
    w, _ = world_rank(group)
    if w > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def max_over_ranks(x: float, device=None, group=None) -> float:
    """max of a host float over ranks (timings are the max over ranks)."""
    w, _ = world_rank(group)
    if w == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sliced_amplitude(contract_range, n_slices: int, group=None, device=None) -> complex:
    """sum_{s} contract(s) over all slices, each rank contracting its block of slices
    (contract_range(lo, hi) -> complex partial sum), summed by one all-reduce."""
    world, rank = world_rank(group)
    lo, hi = block_range(n_slices, world, rank)
    part = contract_range(lo, hi) if hi > lo else 0j
    if world == 1:
        return complex(part)
    t = torch.tensor([part.real, part.imag], dtype=torch.float64, device=device)
    allreduce_sum_(t, group)
    return complex(t[0].item(), t[1].item())


def amplitudes_by_bitstring(contract_one, bits, group=None, device=None):
    """Amplitudes of all bitstrings; rank r contracts its contiguous block
    (contract_one(bitstring) -> complex).  Results are gathered by an all-reduce of
    disjoint supports (not a data-path collective: every amplitude is computed by
    exactly one rank)."""
    n = len(bits)
    world, rank = world_rank(group)
    lo, hi = block_range(n, world, rank)
    mine = torch.zeros(2 * n, dtype=torch.float64, device=device)
    for j in range(lo, hi):
        a = contract_one(bits[j])
        mine[2 * j], mine[2 * j + 1] = a.real, a.imag
    allreduce_sum_(mine, group)
    v = mine.cpu().numpy()
    return v[0::2] + 1j * v[1::2]
