"""Multi-GPU partitioning of the contraction (one process per GPU, torch.distributed).

Two ways the path shards (BASELINE north_star "Index slicing and multi-GPU
partitioning"):
  * bitstrings: independent amplitudes -> contiguous blocks of the batch per rank, no
    data-path collective (an all_gather only returns the results to every rank);
  * slices: the sliced sub-contractions of ONE amplitude ("index
    slicing") are independent -> contiguous slice ranges per rank, the partial
    amplitudes are summed with ONE all-reduce (NCCL over NVLink on the GPU path).
The contraction itself is a callable so the host logic is testable with gloo on CPU.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def block_range(n: int, world: int, rank: int):
    """Contiguous, balanced block [lo, hi) of n items for `rank`."""
    q, r = divmod(n, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def sliced_amplitude(contract_range, n_slices: int, group=None, device=None) -> complex:
    """sum_{s} contract(s) over all slices, each rank contracting its block of slices
    (contract_range(lo, hi) -> complex partial sum), summed by one all-reduce."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = block_range(n_slices, world, rank)
    part = contract_range(lo, hi) if hi > lo else 0j
    if world == 1:
        return complex(part)
    t = torch.tensor([part.real, part.imag], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return complex(t[0].item(), t[1].item())


def amplitudes_by_bitstring(contract_one, bits, group=None, device=None):
    """Amplitudes of all bitstrings; rank r contracts its contiguous block
    (contract_one(bitstring) -> complex).  Results are all-gathered (not a data-path
    collective: every amplitude is computed by exactly one rank)."""
    n = len(bits)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = block_range(n, world, rank)
    mine = torch.zeros(2 * n, dtype=torch.float64, device=device)
    for j in range(lo, hi):
        a = contract_one(bits[j])
        mine[2 * j], mine[2 * j + 1] = a.real, a.imag
    if world > 1:
        dist.all_reduce(mine, op=dist.ReduceOp.SUM, group=group)   # disjoint supports: a gather
    v = mine.cpu().numpy()
    return v[0::2] + 1j * v[1::2]
