#!/usr/bin/env python
"""Benchmark of the contraction hot path (BASELINE.json metric: contraction FLOP/s and
amplitudes/s on B200, % of tensor-pipe peak).

Default workload (N=1): configs[1] -- 8x8 qubit lattice, depth 16, Haar U(2) + CZ
brickwork, complex64 on block-scaled fp16x2 split-precision tensor cores, separator
order (SM Algorithm 1, best of 256 randomized hierarchies) sliced to 2^32-entry tensors.
Its batch of 1024 seeded bitstrings is split into contiguous blocks per rank (weak
scaling, no data-path collective; paper_2208_01498_b200/dist.py).  One STEP = one
contributing slice of one amplitude (the separator tree over one sliced sub-network,
minus its slice-invariant subtrees, which tn_prepare contracts once per bitstring and
keeps); a rank walks its bitstrings, each through its contributing slices.
Intermediates are GBs, far larger than the 126 MB L2, so no L2 flush is needed.

--config 2 / 4 (Sycamore-53 m=14, (2+1)D 12x12 depth 20; complex64): one amplitude,
its contributing slices split into disjoint contiguous blocks per rank, the per-step
partial amplitudes summed over ranks by ONE all-reduce (NCCL) inside the timed region.
--config 3 (IQP 10x10, complex128 on the FP64 tensor pipe): one STEP = one full
amplitude (unsliced), contiguous blocks of the 256 bitstrings per rank.

The timed steps go through tn_prepare / tn_contract_prepared with a profile: each replays
a profiled CUDA graph (the plan's launches with CUDA event records between the kernel
classes) in deferred mode (tn_profile_defer: no wait per call; the device times are
collected by tn_profile_collect after the region); their per-step amplitudes are checked
against the unprofiled CUDA-graph path for the same (bitstring, slice) afterwards.

--impl reference: the oracle (numpy complex128, oracle/) on the host cores, along the
oracle's own order for the workload (oracle/orders/config<C>.json, written by
scripts/write_oracle_orders.py with oracle.ssa.find_order only); it does not load the
product library.

  python bench.py [--gpus N --steps K --warmup W] [--config C] [--impl reference]
Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "contraction FLOP/s"
ORDER_SEED = 0
# per config: arithmetic type, how the units shard across ranks, slicing target (largest
# tensor of a slice 2^t entries, chosen so the plan's arena fits 180 GB), randomized
# separator hierarchies built (the one with the least Eq. (3) work of all slices kept,
# DESIGN.md R10: the slicing overhead differs by orders of magnitude between
# hierarchies), the IQP hyperedge reading R3.  Must equal scripts/write_oracle_orders.py.
SPEC = {
    1: dict(dtype="c64", shard="bits", slice_log=32, hyper=False, n_seeds=256),
    2: dict(dtype="c64", shard="slices", slice_log=33, hyper=False, n_seeds=256),
    3: dict(dtype="c128", shard="bits", slice_log=0, hyper=True, n_seeds=4),
    4: dict(dtype="c64", shard="slices", slice_log=32, hyper=False, n_seeds=1024),
}
ORDERS = os.path.join(ROOT, "oracle", "orders")
TRAFFIC = os.path.join(ROOT, "profiles", "r02", "traffic.json")
# complex128 GEMM on DMMA: MEASURED_PEAKS.json has no fp64 figure; our own probe
# (scripts/probes/dmma_peak.cu, profiles/r01/fp64_tensor_peak.md) measured 37.0 TF/s of
# back-to-back register-only mma.sync f64 on this pool's B200 (burst clock)
FP64_TC_TFLOPS = 37.0
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
# split-precision complex64: one complex MAC (8 useful flops) = 4 real products x 3 fp16
# piece products (hi.hi, hi.lo, lo.hi) = 24 fp16 tensor flops; fp16 dense rate = bf16 rate
F16_FLOPS_PER_USEFUL = 24.0 / 8.0


def load_peaks():
    try:
        return json.load(open(PEAKS_PATH)), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class Clocks:
    """SM clock and clock-event reasons sampled DURING the timed region: an NVML polling
    thread (5 ms period) that has taken its first sample before __enter__ returns, so
    even a region of a few milliseconds gets samples (nvidia-smi -lms needs ~0.1 s to
    start).  Falls back to an nvidia-smi subprocess if NVML is unavailable."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    MASKS = [0x8, 0x40, 0x20, 0x4]      # nvmlClocksEventReason{HwSlowdown,HwThermalSlowdown,SwThermalSlowdown,SwPowerCap}

    def __init__(self, index=0, period_s=0.005):
        self.index = index
        self.period = period_s
        self.rows = []                  # (sm_mhz, max_mhz, reasons bitmask[, board power W])
        self.limit_w = None
        self.proc = None
        self.stop = threading.Event()
        self.t = None

    def _poll(self, nv, h, first):
        while True:
            try:
                self.rows.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                                  float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)),
                                  int(nv.nvmlDeviceGetCurrentClocksEventReasons(h)),
                                  nv.nvmlDeviceGetPowerUsage(h) / 1000.0))
                if self.limit_w is None:
                    self.limit_w = nv.nvmlDeviceGetEnforcedPowerLimit(h) / 1000.0
            except Exception:
                pass
            first.set()
            if self.stop.wait(self.period):
                return

    def _handle(self, nv):
        # the CUDA device's own NVML handle by PCI address (NVML enumerates every GPU of the
        # machine regardless of CUDA_VISIBLE_DEVICES), else by index
        try:
            import torch
            p = torch.cuda.get_device_properties(self.index)
            bus = "%08x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
            return nv.nvmlDeviceGetHandleByPciBusId(bus.encode() if isinstance(bus, str) else bus)
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.index)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = self._handle(nv)
            first = threading.Event()
            self.t = threading.Thread(target=self._poll, args=(nv, h, first), daemon=True)
            self.t.start()
            first.wait(2.0)
            return self
        except Exception:
            self.t = None
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            r = [v.strip() for v in line.split(",")]
            if len(r) >= 6 and r[0].replace(".", "").isdigit() and r[1].replace(".", "").isdigit():
                mask = sum(m for m, v in zip(self.MASKS, r[2:6]) if v == "Active")
                self.rows.append((float(r[0]), float(r[1]), mask))

    def __exit__(self, *a):
        if self.t is not None:
            self.stop.set()
            self.t.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = list(self.rows)
        sm = [r[0] for r in rows]
        reasons = sorted({n for r in rows for n, m in zip(self.NAMES, self.MASKS) if r[2] & m})
        pw = [r[3] for r in rows if len(r) > 3]
        out = {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(r[1] for r in rows) if rows else None,
               "reasons": reasons, "samples": len(rows), "sampler": "nvml" if self.t is not None else "nvidia-smi"}
        if pw:
            out["power_w"] = float(np.median(pw))
            out["power_limit_w"] = self.limit_w
        return out


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload(ci):
    from tn_inputs import config_circuit, random_bitstrings, CONFIGS
    c = config_circuit(ci)
    bits = random_bitstrings(c.n, max(1, CONFIGS[ci]["n_bitstrings"]), 1)
    return c, bits


def oracle_order(ci):
    """The workload's separator order as the ORACLE found it (oracle/orders/, written by
    scripts/write_oracle_orders.py; tn_find_order reproduces it bit for bit,
    tests/test_library_host.py)."""
    path = os.path.join(ORDERS, f"config{ci}.json")
    with open(path) as f:
        o = json.load(f)
    spec = SPEC[ci]
    assert (o["seed"], o["n_seeds"], o["max_log2_size"], o["diag_hyper"]) == \
        (ORDER_SEED, spec["n_seeds"], spec["slice_log"], spec["hyper"]), f"{path} does not match SPEC[{ci}]"
    return o


def workload_name(ci, c):
    spec = SPEC[ci]
    return (f"configs[{ci}]: {c.name}; separator order seed {ORDER_SEED}, best of {spec['n_seeds']} randomized "
            f"hierarchies" + (f"; slicing to 2^{spec['slice_log']}-entry tensors" if spec["slice_log"] else ""))


def shared_config(ci, c, n_bits, slice_bits, flops_slice):
    """`config` of the JSON line, identical for both arms: the workload, what one step
    is, and its Eq. (3) flops (8 M per pairwise step, R13) -- all fixed by the circuit and
    the order, none by the implementation."""
    spec = SPEC[ci]
    if spec["shard"] == "slices":
        step = (f"one contributing slice (of 2^{slice_bits}) of one amplitude; ranks take disjoint contiguous blocks "
                f"of its slices, per-step partial amplitudes summed by one all-reduce in the timed region")
    elif slice_bits:
        step = (f"one contributing slice (of 2^{slice_bits}) of one amplitude; the batch of {n_bits} bitstrings in "
                f"contiguous blocks per rank, each bitstring through its contributing slices")
    else:
        step = f"one full amplitude (unsliced); the batch of {n_bits} bitstrings in contiguous blocks per rank"
    return {"workload": workload_name(ci, c), "step": step, "flops_per_step": flops_slice, "slice_bits": slice_bits,
            "l2": "working set (intermediates of GBs) >> 126 MB L2, no flush between steps"}


def oracle_flops_per_slice(net, o):
    """8 x (Eq. (3) multiplications of one slice) from the oracle's own order."""
    from oracle.ssa import sliced_work
    return 8.0 * sliced_work(net, [tuple(p) for p in o["steps"]], o["slices"]) / 2.0 ** o["slice_bits"]


def cpu_baseline_sample(c, bits, o, budget_s=15.0, hyper=False):
    """The oracle as it stands on the host cores: slice 0 of bitstring 0 along the
    oracle's own order (oracle/orders/), contracting the steps of the separator tree in
    order with oracle.contract.contract_pair (numpy complex128) until `budget_s` of
    wall time; FLOP/s = sum 8 M / elapsed.  Steps too large for the budget (M > 2^33)
    and the steps depending on them are skipped."""
    from oracle.network import build_network
    from oracle.contract import kept_per_step, leaf_tensors, contract_pair
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    net = build_network(c, diag_hyper=hyper)
    steps = [tuple(p) for p in o["steps"]]
    sl = o["slices"]
    kept = kept_per_step(net, steps)
    fixed = {i: 0 for i in sl}
    n = len(net.tensors)
    nodes = dict(enumerate(leaf_tensors(net, bits[0], fixed)))
    flops = 0.0
    done = 0
    skipped = 0
    t0 = time.perf_counter()
    for k, (a, b) in enumerate(steps):
        if a not in nodes or b not in nodes:       # depends on a skipped step
            nodes.pop(a, None), nodes.pop(b, None)
            skipped += 1
            continue
        (Ai, A), (Bi, B) = nodes[a], nodes[b]
        uni = (set(Ai) | set(Bi)) - set(fixed)
        m = sum(int(math.log2(net.dims[i])) for i in uni)
        nodes.pop(a), nodes.pop(b)
        if m > 33:        # bounded sample: steps too large for the CPU budget are skipped
            skipped += 1
            continue
        kk = [i for i in kept[k] if i not in fixed]
        nodes[n + k] = contract_pair(Ai, A, Bi, B, kk, net.dims)
        flops += 8.0 * 2.0 ** m
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    el = time.perf_counter() - t0
    return {"value": flops / el, "unit": "FLOP/s", "cores": int(cores), "kind": "oracle", "elapsed_s": el,
            "sample": f"oracle (numpy complex128, plain einsum pairs) on slice 0 of bitstring 0 along the oracle's "
                      f"own order: {done} of the {len(steps)} pairwise steps in order, skipping {skipped} with "
                      f"M > 2^33 or depending on one ({flops:.3g} flops, {el:.1f} s)"}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    spec = SPEC[args.config]
    c, bits = workload(args.config)
    from oracle.network import build_network
    o = oracle_order(args.config)
    net = build_network(c, diag_hyper=spec["hyper"])
    cfg = shared_config(args.config, c, len(bits), o["slice_bits"], oracle_flops_per_slice(net, o))
    vals = []
    for _ in range(args.warmup + args.steps):
        vals.append(cpu_baseline_sample(c, bits, o, budget_s=max(2.0, 60.0 / (args.warmup + args.steps)),
                                        hyper=spec["hyper"]))
    timed = vals[args.warmup:]
    v = float(np.mean([t["value"] for t in timed]))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "FLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(np.mean([t["elapsed_s"] for t in timed])), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic", "config": cfg,
            "arithmetic": "numpy complex128 on the host (the oracle); each step a bounded sample of the workload's "
                          "step (cpu_baseline.sample)",
            "cpu_baseline": {"value": v, "unit": "FLOP/s", "cores": timed[0]["cores"], "kind": "oracle",
                             "sample": timed[0]["sample"]},
            "e2e": {"value": v, "unit": "FLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def load_traffic(ci):
    """DRAM traffic of the dominant kernel per launch from a committed ncu --set full
    capture (profiles/r02/traffic.json, written by scripts/traffic_from_ncu.py)."""
    try:
        return json.load(open(TRAFFIC)).get(f"config{ci}")
    except Exception:
        return None


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    # under torchrun (WORLD_SIZE set) the process group exists even for one rank, so the
    # NCCL paths (barrier, slice all-reduce, max-over-ranks timing) run at every N
    distributed = "WORLD_SIZE" in os.environ
    if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION"):
        os.environ["NCCL_DEBUG"] = "WARN"      # keep stdout to the one JSON line (no version banner)
    if distributed:
        import torch.distributed as tdist
        # rank 0 alone runs the host order search (all cores) and broadcasts it
        # (dist.shared_order); a long search must not trip the collective timeout
        import datetime
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local), timeout=datetime.timedelta(hours=2))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2208_01498_b200 as tb
    from paper_2208_01498_b200 import dist as pdist

    ci = args.config
    spec = SPEC[ci]
    c, bits = workload(ci)
    dtype = tb.TN_C64 if spec["dtype"] == "c64" else tb.TN_C128
    net = tb.Network.from_circuit(c, diag_hyper=spec["hyper"])
    order = pdist.shared_order(
        lambda: tb.Order(net, seed=ORDER_SEED, n_seeds=spec["n_seeds"], max_log2_size=spec["slice_log"]),
        lambda st, sl, mf: tb.Order.from_steps(net, st, sl, mf), device=dev)
    oinfo = order.info()
    plan = tb.Plan(net, order, dtype=dtype, device=local)      # raises if the arena does not fit
    pinfo = plan.info()
    n_slices = int(pinfo["n_slices"])
    slice_bits = int(pinfo["slice_bits"])
    flops_slice = float(pinfo["flops_per_slice"])
    by_slices = spec["shard"] == "slices"
    K, W = args.steps, args.warmup
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream

    # ---- work items (row of the batch, slice id): one per step, from dist.py ----
    if by_slices:
        live = plan.contributing_slice_ids(bits[0], 0, ws * K)
        mine = pdist.slice_block(live, ws, rank)
        if not mine:
            raise RuntimeError(f"rank {rank}: no slice to contract ({len(live)} contributing slices for {ws} ranks)")
        items = [(0, s) for s in mine]
        warm = [items[j % len(items)] for j in range(W)]
    else:
        lo, hi = pdist.block_range(len(bits), ws, rank)
        rows = list(range(lo, hi))
        if n_slices > 1:
            items = pdist.bitstring_steps(lambda r, n: plan.contributing_slice_ids(bits[r], 0, n), rows, K + W)
        else:
            items = [(r, 0) for r in rows[:K + W]]
        if len(items) < K + W:
            raise RuntimeError(f"rank {rank}: {len(items)} work items for {K + W} steps")
        warm, items = items[K:], items[:K]
    steps_mine = len(items)
    bits_dev = torch.from_numpy(np.ascontiguousarray(bits)).to(dev)
    # one complex128 accumulator per step (the same length K on every rank: the all-reduce of
    # the sliced configs sums them elementwise over ranks)
    amp = torch.zeros(max(K, 1), dtype=torch.complex128, device=dev)
    scratch = torch.zeros(1, dtype=torch.complex128, device=dev)

    flops_pro = float(pinfo["flops_prologue"])          # slice-invariant part, once per bitstring
    flops_dep = flops_slice - flops_pro                   # the rest, once per slice

    def run(work, amps, profiled, ev=None):
        """contract `work` (row, slice) items: tn_prepare (the bitstring's slice-invariant
        prologue) whenever the row changes, tn_contract_prepared per slice into amps[j];
        returns (profiles, prologues run).  ev: lists of CUDA events around the calls."""
        cur, n_pre, profs = None, 0, []
        for j, (row, s) in enumerate(work):
            if row != cur:
                if ev is not None:
                    ev["pro"].append((torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)))
                    ev["pro"][-1][0].record(stream)
                profs.append(plan.prepare(bits_dev[row].data_ptr(), sptr, profiled=profiled))
                if ev is not None:
                    ev["pro"][-1][1].record(stream)
                cur, n_pre = row, n_pre + 1
            if ev is not None:
                ev["slice"].append((torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)))
                ev["slice"][-1][0].record(stream)
            profs.append(plan.contract_prepared(s, s + 1, amps[j:j + 1].data_ptr(), sptr, profiled=profiled))
            if ev is not None:
                ev["slice"][-1][1].record(stream)
        return profs, n_pre

    run(warm, scratch.expand(max(len(warm), 1)), False)
    torch.cuda.synchronize()

    def barrier():
        if distributed:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # ---- timed region: the steps through the profiled launchers (+ the slice all-reduce) ----
    launches0 = tb.kernel_launches()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev = {"pro": [], "slice": []}
    # profiled calls in deferred mode: each replays a profiled CUDA graph without waiting
    # for it (the per-kernel-class device times are collected after the region), so the
    # host keeps the GPU fed as in the unprofiled graph path
    plan.profile_defer(True)
    with Clocks(local) as clk:
        e0.record(stream)
        profs, n_pre = run(items, amp, True, ev)
        if by_slices:
            amp_mine = amp.clone()                  # (this rank's values, for the check below)
            pdist.allreduce_sum_(amp)               # partial amplitudes of all ranks' slices
        e1.record(stream)
        barrier()
    profs.append(plan.profile_collect())            # the device times of the deferred replays
    plan.profile_defer(False)
    launches = tb.kernel_launches() - launches0
    prof = profs[0]
    for p in profs[1:]:
        for k, v in p.items():
            if k == "kernels":
                for name, d in v.items():
                    for f, x in d.items():
                        prof["kernels"][name][f] += x
            else:
                prof[k] += v
    ms = pdist.max_over_ranks(e0.elapsed_time(e1), dev)
    flops_mine = n_pre * flops_pro + steps_mine * flops_dep        # executed flops of this rank
    t_fl = torch.tensor([flops_mine], dtype=torch.float64, device=dev)
    pdist.allreduce_sum_(t_fl)
    total_flops = float(t_fl.item())
    value = total_flops / (ms / 1e3)
    t_pro = float(np.mean([a.elapsed_time(b) for a, b in ev["pro"]])) / 1e3
    t_slice = float(np.mean([a.elapsed_time(b) for a, b in ev["slice"]])) / 1e3

    # ---- the timed amplitudes against the CUDA-graph path (same bitstring and slice) ----
    n_chk = min(steps_mine, 2)
    chk = torch.zeros(max(n_chk, 1), dtype=torch.complex128, device=dev)
    run(items[:n_chk], chk, False)
    torch.cuda.synchronize()
    a_t, a_g = (amp_mine if by_slices else amp)[:n_chk].cpu().numpy(), chk[:n_chk].cpu().numpy()
    rel = float(np.max(np.abs(a_t - a_g) / np.maximum(np.abs(a_g), 1e-300))) if n_chk else 0.0
    if not rel <= 1e-9:
        raise RuntimeError(f"timed (profiled) amplitudes differ from the graph path: {a_t} vs {a_g}")

    # amplitudes/s: an amplitude = its prologue + its contributing slices (provably zero
    # ones are skipped by tn_contract / tn_amplitudes; mean count over the whole batch),
    # timed on the device in the timed region (max over ranks)
    if n_slices > 1:
        contrib_mean = float(np.mean([plan.contributing_slices(b) for b in bits]))
    else:
        contrib_mean = 1.0
    t_amp = pdist.max_over_ranks(t_pro + contrib_mean * t_slice, dev)
    amps_per_s = ws / t_amp

    # ---- e2e: the public host-buffer call, H2D bits (pinned host memory) + D2H amplitude
    # inside the region ----
    e2e_items = items[:max(1, min(K, 3))]
    pinned = torch.from_numpy(np.ascontiguousarray(bits)).pin_memory().numpy()
    barrier()
    t0 = time.perf_counter()
    for row, s in e2e_items:
        plan.contract(pinned[row], s, s + 1)
    barrier()
    e2e_s = pdist.max_over_ranks(time.perf_counter() - t0, dev)
    e2e_value = flops_slice * len(e2e_items) * ws / e2e_s       # each call: prologue + one slice

    # ---- unsliced bitstring configs: throughput of tn_amplitudes with concurrent lanes ----
    lanes_line = None
    if not by_slices and n_slices == 1:
        try:
            plan.set_lanes(4)
            lo, hi = pdist.block_range(len(bits), ws, rank)
            batch = np.ascontiguousarray(bits[lo:hi])
            plan.amplitudes(batch[:8])
            dts = []
            for _ in range(3):                  # median of 3 calls over this rank's whole batch
                barrier()
                t0 = time.perf_counter()
                plan.amplitudes(batch)
                barrier()
                dts.append(pdist.max_over_ranks(time.perf_counter() - t0, dev))
            dt_l = float(np.median(dts))
            lanes_line = {"lanes": 4, "amplitudes": int(len(batch)) * ws, "value": len(batch) * ws / dt_l,
                          "unit": "amplitudes/s", "call": "tn_amplitudes (host bitstrings in, host amplitudes out), "
                                                          "median of 3 calls"}
        except tb.TnError as e:
            print(f"lanes: {e}", file=sys.stderr)

    if rank != 0:
        if distributed:
            torch.distributed.destroy_process_group()
        return 0
    peaks, peak_src = load_peaks()
    sustained = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    hbm = peaks["hbm_gbs"]
    if dtype == tb.TN_C64:
        peak_tc = sustained / F16_FLOPS_PER_USEFUL
        tc_note = (f"{peak_src} bf16 sustained {sustained} TF/s (= fp16 dense rate) x 8/24 (useful complex flops per "
                   "fp16 tensor flop of the fp16x2 scheme)")
    else:
        peak_tc = FP64_TC_TFLOPS
        tc_note = ("fp64 tensor peak 37.0 TF/s measured by scripts/probes/dmma_peak.cu (register-only mma.sync f64, "
                   "burst clock; profiles/r01/fp64_tensor_peak.md); complex128 flops are executed flops")
    tensor_classes = {"cgemm_f16x2s_kernel", "cgemm2_f16x2s_kernel", "cgemm2p_f16x2s_kernel", "zgemm_dmma_kernel"}
    hbm_classes = {"small_contract_kernel", "pack_f16x2s_kernel", "pack_planar_kernel", "skinny_kernel", "wide_kernel"}
    kern = {}
    for name, d in prof["kernels"].items():
        if d["ms"] <= 0:
            continue
        r = {"ms": d["ms"], "share_of_step": d["ms"] / ms}
        if name in tensor_classes and d["flops"] > 0:
            r.update(achieved=d["flops"] / (d["ms"] / 1e3) / 1e12, unit="TFLOP/s", peak=peak_tc)
        elif name in hbm_classes and d["bytes"] > 0:
            r.update(achieved=d["bytes"] / (d["ms"] / 1e3) / 1e9, unit="GB/s", peak=hbm)
        if "achieved" in r:
            r["frac"] = r["achieved"] / r["peak"]
        kern[name] = r
    dom = max((k for k in kern if "achieved" in kern[k]), key=lambda k: kern[k]["ms"])
    dk = kern[dom]
    roof = {"bound": "tensor" if dom in tensor_classes else "hbm", "achieved": dk["achieved"], "peak": dk["peak"],
            "unit": dk["unit"], "frac": dk["frac"], "traffic": None, "kernel": dom, "share_of_step": dk["share_of_step"],
            "peak_note": tc_note if dom in tensor_classes else f"{peak_src} HBM copy bandwidth (read + write bytes)",
            "achieved_note": "algorithmic flops (8 M per step, R13) or bytes (DESIGN.md Kernels) of every launch of "
                             "this kernel class / its summed CUDA-event time on the launching stream"}
    tr = load_traffic(ci)
    if tr and tr.get("kernel") == dom:
        roof["traffic"] = tr["dram_bytes"]
        roof["traffic_probe"] = tr
    clocks = clk.summary()
    if roof["bound"] == "tensor" and dtype == tb.TN_C64 and clocks.get("sm_mhz"):
        # the measured cuBLAS "sustained" denominator ran at its own power-capped clock; the
        # tensor pipe's own ceiling at this run's median clock: a 128 x 128 x 16 tcgen05 MMA
        # every 64 cycles per SM (8192 fp16 flops / clk / SM), 24 fp16 flops per useful 8
        at_clk = 8192.0 * 148 * clocks["sm_mhz"] * 1e6 / 1e12 / F16_FLOPS_PER_USEFUL
        roof["clock_ceiling"] = {"sm_mhz": clocks["sm_mhz"], "useful_tflops": at_clk, "frac": roof["achieved"] / at_clk,
                                 "note": "8192 fp16 flops/clk/SM (tcgen05 m128n128k16 floor of 64 cycles) x 148 SMs "
                                         "x median SM clock of the timed region / 3"}
    line = {
        "metric": METRIC, "value": value, "unit": "FLOP/s", "n_gpus": ws, "steps": K,
        "warmup": W, "ms_per_step": ms / max(steps_mine, 1), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": spec["dtype"], "data": "synthetic",
        "config": shared_config(ci, c, len(bits), slice_bits, flops_slice),
        "arithmetic": ("complex64 on block-scaled fp16x2 split-precision tcgen05 tensor cores (fp32 accumulation), "
                       "CUDA-core fp32 for skinny / wide steps" if dtype == tb.TN_C64 else
                       "complex128 on the FP64 tensor pipe (DMMA) and fp64 CUDA cores"),
        "amplitudes_per_s": amps_per_s,
        "contributing_slices_mean": contrib_mean,
        "executed_flops_per_step": flops_mine / max(steps_mine, 1),
        "slice_reuse": {"prologue_flops_fraction_of_slice": flops_pro / flops_slice,
                        "frontier_gb": pinfo["frontier_bytes"] / 1e9, "prologues_timed": n_pre,
                        "t_prologue_s": t_pro, "t_slice_s": t_slice,
                        "note": "the slice-invariant subtrees are contracted once per bitstring (tn_prepare) and "
                                "kept while its slices run (tn_contract_prepared); value = executed flops / time; "
                                "amplitudes_per_s = N / (t_prologue + contributing_slices_mean x t_slice)"},
        "amplitudes_per_s_lanes": lanes_line,
        "slicing": {"slice_bits": slice_bits, "log2_sliced_work": oinfo["log2_slice_2M"] - 1.0 + slice_bits,
                    "log2_unsliced_work": oinfo["log2_total_2M"] - 1.0,
                    "note": "Eq. (3) multiplications sum_k M_k of the whole amplitude: all slices vs the unsliced "
                            "order (the slicing overhead)",
                    "ssa_splits_median_fallbacks": oinfo["median_fallbacks"]},
        "plan": {"arena_gb": pinfo["arena_bytes"] / 1e9, "tc_flops_fraction": pinfo["tc_flops_per_slice"] / flops_slice,
                 "launches_per_slice": pinfo["n_launches_per_slice"]},
        "roofline": roof,
        "kernels": kern,
        "check": {"steps": n_chk, "max_rel_diff_vs_graph_path": rel},
        "e2e": {"value": e2e_value, "unit": "FLOP/s", "h2d_bytes_per_step": int(c.n), "d2h_bytes_per_step": 16},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if not args.no_cpu_baseline and ws == 1:      # the oracle baseline: rank 0 at N = 1 only
        line["cpu_baseline"] = cpu_baseline_sample(c, bits, oracle_order(ci), budget_s=args.cpu_budget,
                                                   hyper=spec["hyper"])
    print(json.dumps(line))
    if distributed:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1, choices=sorted(SPEC))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    args = ap.parse_args()
    # stdout carries exactly one JSON line: Python's prints go to the original stdout, while
    # file descriptor 1 (native libraries: NCCL's version banner under torchrun) goes to stderr
    real_out = os.dup(1)
    os.dup2(2, 1)
    sys.stdout = os.fdopen(real_out, "w", buffering=1)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
