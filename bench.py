#!/usr/bin/env python
"""Benchmark of the contraction hot path (BASELINE.json metric: contraction FLOP/s and
amplitudes/s on B200, % of tensor-pipe peak).

Default workload (N=1): configs[1] -- 8x8 qubit lattice, depth 16, Haar U(2) + CZ
brickwork, complex64 on block-scaled fp16x2 split-precision tensor cores, separator
order (SM Algorithm 1) sliced so every tensor fits HBM.  Its amplitudes are partitioned
by bitstring across ranks (weak scaling): rank r contracts bitstrings r, r+N, ... of the
seeded batch of 1024.  One STEP = one slice of one amplitude (the whole separator tree
over one sliced sub-network); an amplitude is n_slices steps.  Intermediates are GBs,
far larger than the 126 MB L2, so no L2 flush is needed between steps.

--config 2 / 4 (Sycamore-53 m=14, (2+1)D 12x12 depth 20; complex64): one amplitude,
its slices partitioned across ranks (rank r takes slices [r K, (r+1) K) of the K timed
steps), the per-rank partial amplitudes summed by ONE NCCL all-reduce inside the timed
region.  --config 3 (IQP 10x10, complex128 on the FP64 tensor pipe): one STEP = one
full amplitude (unsliced), bitstrings r::N of 256 per rank.

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
# per config: arithmetic type, how the units shard across ranks, slicing targets tried in
# order (largest tensor of a slice 2^t entries; the first plan that fits HBM is used)
# n_seeds: randomized separator hierarchies built, the one with the least Eq. (3) work of
# all slices kept (R10) -- for sliced configs the slicing overhead varies by
# orders of magnitude between hierarchies (configs[1]: 2^59.2 with 4, 2^56.7 with 64,
# 2^54.6 with 256; built on host threads, ~10 s)
SPEC = {
    1: dict(dtype="c64", shard="bits", slice_logs=(34, 33, 32, 31), hyper=False, n_seeds=256),
    2: dict(dtype="c64", shard="slices", slice_logs=(34, 33, 32, 31), hyper=False, n_seeds=256),
    3: dict(dtype="c128", shard="bits", slice_logs=(0,), hyper=True, n_seeds=4),
    4: dict(dtype="c64", shard="slices", slice_logs=(34, 33, 32, 31), hyper=False, n_seeds=1024),
}
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


def cpu_baseline_sample(c, bits, steps, sl, budget_s=15.0, hyper=False):
    """The oracle as it stands on the host cores: slice 0 of bitstring 0 of the same
    network and the same order (the step list and sliced indices of the plan, from
    tn_find_order -- the oracle's own find_order builds the identical order, bit for
    bit, but takes minutes in Python for 64 hierarchies), contracting the steps of the
    separator tree in order with oracle.contract.contract_pair until `budget_s` of CPU
    time; FLOP/s = sum 8 M / elapsed."""
    from oracle.network import build_network
    from oracle.contract import kept_per_step, leaf_tensors, contract_pair
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    net = build_network(c, diag_hyper=hyper)
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
            "sample": f"oracle (numpy complex128) on slice 0 of bitstring 0: {done} of the {len(steps)} pairwise "
                      f"steps of the separator tree in order, skipping {skipped} steps with M > 2^33 or depending on "
                      f"one ({flops:.3g} flops, {el:.1f} s)"}


def workload_name(ci, c, slice_log2):
    spec = SPEC[ci]
    prec = "block-scaled fp16x2 split on tcgen05" if spec["dtype"] == "c64" else "FP64 tensor pipe (DMMA)"
    return (f"configs[{ci}]: {c.name}; {spec['dtype']} ({prec}); separator order seed {ORDER_SEED}, "
            f"best of {spec['n_seeds']} randomized hierarchies"
            + (f"; slicing to 2^{slice_log2}-entry tensors" if slice_log2 else ""))


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    spec = SPEC[args.config]
    c, bits = workload(args.config)
    import paper_2208_01498_b200 as tb       # host-only calls: network + order (no device)
    net = tb.Network.from_circuit(c, diag_hyper=spec["hyper"])
    order = tb.Order(net, seed=ORDER_SEED, n_seeds=spec["n_seeds"], max_log2_size=spec["slice_logs"][0])
    vals = []
    for _ in range(args.warmup + args.steps):
        vals.append(cpu_baseline_sample(c, bits, order.steps(), order.slices(),
                                        budget_s=max(2.0, 60.0 / (args.warmup + args.steps)), hyper=spec["hyper"]))
    timed = vals[args.warmup:]
    v = float(np.mean([t["value"] for t in timed]))
    cfg = {"workload": workload_name(args.config, c, spec["slice_logs"][0]),
           "step": "a bounded sample of one slice's pairwise steps (see cpu_baseline.sample)"}
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "FLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(np.mean([t["elapsed_s"] for t in timed])), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": v, "unit": "FLOP/s", "cores": timed[0]["cores"], "kind": "oracle",
                             "sample": timed[0]["sample"]},
            "e2e": {"value": v, "unit": "FLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    # under torchrun (WORLD_SIZE set) the process group exists even for one rank, so the
    # NCCL paths (barrier, slice all-reduce, max-over-ranks timing) run at every N
    distributed = "WORLD_SIZE" in os.environ
    if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION"):
        os.environ["NCCL_DEBUG"] = "WARN"      # keep stdout to the one JSON line (no version banner)
    if distributed:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2208_01498_b200 as tb

    ci = args.config
    spec = SPEC[ci]
    c, bits = workload(ci)
    dtype = tb.TN_C64 if spec["dtype"] == "c64" else tb.TN_C128
    net = tb.Network.from_circuit(c, diag_hyper=spec["hyper"])
    plan = None
    for slice_log2 in spec["slice_logs"]:
        order = tb.Order(net, seed=ORDER_SEED, n_seeds=spec["n_seeds"], max_log2_size=slice_log2)
        try:
            plan = tb.Plan(net, order, dtype=dtype, device=local)
            break
        except tb.TnError as e:       # arena does not fit this GPU: slice further
            print(f"slicing target 2^{slice_log2}: {e}", file=sys.stderr)
    if plan is None:
        raise RuntimeError("no slicing target fits device memory")
    pinfo = plan.info()
    n_slices = int(pinfo["n_slices"])
    slice_bits = int(pinfo["slice_bits"])
    flops_slice = float(pinfo["flops_per_slice"])
    by_slices = spec["shard"] == "slices"
    # one step: one slice (sliced configs) or one whole amplitude (unsliced)
    step_slices = 1 if n_slices > 1 else n_slices
    my_bits = bits[0:1] if by_slices else bits[rank::ws]
    bits_dev = torch.from_numpy(np.ascontiguousarray(my_bits)).to(dev)
    nq = c.n
    amp = torch.zeros(1, dtype=torch.complex128, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream

    # steps run contributing slices only (provably zero ones are skipped by tn_contract /
    # tn_amplitudes, so they are not work an amplitude needs)
    total_steps = args.steps + args.warmup
    if by_slices:       # rank r: contributing slices [r K, (r + 1) K) of one amplitude, then warm-ups
        live = plan.contributing_slice_ids(my_bits[0], 0, (ws + 1) * total_steps)
        mine = live[rank * args.steps:(rank + 1) * args.steps] + live[ws * args.steps:ws * args.steps + args.warmup]
    elif n_slices > 1:  # config 1: contributing slices of this rank's first bitstring
        mine = plan.contributing_slice_ids(my_bits[0], 0, total_steps)
    else:
        mine = [0]
    mine = (mine * (total_steps // max(len(mine), 1) + 1))[:total_steps]

    def step_args(j):
        """(bitstring row, first slice) of this rank's j-th step (j >= steps: warm-ups)"""
        if n_slices > 1:
            return 0, mine[j]
        return j % len(my_bits), 0

    for w in range(args.warmup):
        row, sl = step_args(args.steps + w)
        plan.contract_device(bits_dev[row].data_ptr(), sl, sl + step_slices, amp.data_ptr(), sptr)
    torch.cuda.synchronize()

    def barrier():
        if distributed:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # ---- timed region: K steps through the profiled launcher (+ the slice all-reduce) ----
    amp.zero_()
    launches0 = tb.kernel_launches()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record(stream)
        prof = {}
        for j in range(args.steps):
            row, sl = step_args(j)
            p = plan.contract_profiled(bits_dev[row].data_ptr(), sl, sl + step_slices, amp.data_ptr(), sptr)
            for k, v in p.items():
                prof[k] = prof.get(k, 0) + v
        if by_slices and distributed:
            torch.distributed.all_reduce(amp)        # partial amplitudes of all ranks' slices
        e1.record(stream)
        barrier()
    launches = tb.kernel_launches() - launches0
    ms = e0.elapsed_time(e1)
    t_max = torch.tensor([ms], dtype=torch.float64, device=dev)
    if distributed:
        torch.distributed.all_reduce(t_max, op=torch.distributed.ReduceOp.MAX)
    ms = float(t_max.item())
    flops_step = flops_slice * step_slices
    total_flops = flops_step * args.steps * ws
    value = total_flops / (ms / 1e3)
    # an amplitude = its contributing slices (provably zero ones are skipped by
    # tn_contract / tn_amplitudes); this rank's first bitstring
    contrib = plan.contributing_slices(my_bits[0]) if n_slices > 1 else 1
    amps_per_s = value / (flops_slice * contrib)

    # ---- e2e: the public host-buffer call, H2D bits (pinned host memory) + D2H amplitude
    # inside the region ----
    e2e_steps = max(1, min(args.steps, 3))
    pinned = torch.from_numpy(np.ascontiguousarray(my_bits)).pin_memory().numpy()
    barrier()
    t0 = time.perf_counter()
    for j in range(e2e_steps):
        row, sl = step_args(j)
        plan.contract(pinned[row], sl, sl + step_slices)
    barrier()
    e2e_s = time.perf_counter() - t0
    t_e = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if distributed:
        torch.distributed.all_reduce(t_e, op=torch.distributed.ReduceOp.MAX)
    e2e_value = flops_step * e2e_steps * ws / float(t_e.item())

    # ---- unsliced bitstring configs: throughput of tn_amplitudes with concurrent lanes ----
    lanes_line = None
    if not by_slices and n_slices == 1:
        try:
            plan.set_lanes(4)
            batch = np.ascontiguousarray(my_bits[:64])
            plan.amplitudes(batch[:8])
            barrier()
            t0 = time.perf_counter()
            plan.amplitudes(batch)
            barrier()
            dt_l = time.perf_counter() - t0
            t_l = torch.tensor([dt_l], dtype=torch.float64, device=dev)
            if distributed:
                torch.distributed.all_reduce(t_l, op=torch.distributed.ReduceOp.MAX)
            lanes_line = {"lanes": 4, "amplitudes": int(len(batch)) * ws, "value": len(batch) * ws / float(t_l.item()),
                          "unit": "amplitudes/s", "call": "tn_amplitudes (host bitstrings in, host amplitudes out)"}
        except tb.TnError as e:
            print(f"lanes: {e}", file=sys.stderr)

    if rank != 0:
        if distributed:
            torch.distributed.destroy_process_group()
        return 0
    peaks, peak_src = load_peaks()
    sustained = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    if dtype == tb.TN_C64:
        peak_tc = sustained / F16_FLOPS_PER_USEFUL
        kname, pnote = "cgemm_f16x2s_kernel (tcgen05)", (
            f"{peak_src} bf16 sustained {sustained} TF/s (= fp16 dense rate) x 8/24 (useful complex flops per "
            "fp16 tensor flop of the fp16x2 scheme)")
    else:
        peak_tc = FP64_TC_TFLOPS
        kname, pnote = "zgemm_dmma_kernel (FP64 tensor pipe, complex128)", (
            "fp64 tensor peak 37.0 TF/s measured by scripts/probes/dmma_peak.cu (register-only mma.sync f64, "
            "burst clock; profiles/r01/fp64_tensor_peak.md); complex128 flops are executed flops")
    gemm_tfs = prof["flops_gemm"] / (prof["ms_gemm"] / 1e3) / 1e12 if prof.get("ms_gemm") else 0.0
    small_gbs = prof["bytes_small"] / (prof["ms_small"] / 1e3) / 1e9 if prof.get("ms_small") else 0.0
    if prof.get("ms_gemm", 0) >= prof.get("ms_small", 0):
        roof = {"bound": "tensor", "achieved": gemm_tfs, "peak": peak_tc, "unit": "TFLOP/s",
                "frac": gemm_tfs / peak_tc if peak_tc else None, "traffic": None, "kernel": kname,
                "peak_note": pnote, "share_of_step": prof["ms_gemm"] / ms if ms else None}
        if dtype == tb.TN_C64:
            # DRAM traffic (bytes) of one launch of the bench's dominant GEMM shape from the
            # committed ncu --set full capture: a K-slab of the (18, 12, 16) steps (64% of a
            # configs[1] step).  A is re-read ~5x from DRAM (L2 hit 78%), harmless for a
            # tensor-bound kernel (DRAM at 13%)
            roof["traffic"] = 5.025e10 + 8.661e9
            roof["traffic_probe"] = {"launch": "cgemm2_f16x2s_kernel, C[2^18][2^12] = A[2^18][2^12] B[2^12][2^12] "
                                               "(one K-slab of the configs[1] (18, 12, 16) steps)",
                                     "dram_bytes": 5.025e10 + 8.661e9, "algorithmic_bytes": 1.731e10,
                                     "tensor_active": 0.930, "source": "profiles/r01/ncu_full_summary.md",
                                     "note": "A panels re-read ~5x from DRAM (L2 hit 78%); the kernel is tensor-bound "
                                             "(DRAM 11% busy) but power-capped, so raster groups / serpentine order / "
                                             "K-chunks were tuned to cut these bytes (DESIGN.md)"}
    else:
        roof = {"bound": "hbm", "achieved": small_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": small_gbs / peaks["hbm_gbs"], "traffic": None, "kernel": "small_contract_kernel",
                "peak_note": f"{peak_src} HBM copy bandwidth; algorithmic bytes = operands + results of each wave",
                "share_of_step": prof["ms_small"] / ms if ms else None}
    clocks = clk.summary()
    if roof["bound"] == "tensor" and dtype == tb.TN_C64 and clocks.get("sm_mhz"):
        # the measured cuBLAS "sustained" denominator ran at its own power-capped clock; the
        # tensor pipe's own ceiling at this run's median clock: a 128 x 128 x 16 tcgen05 MMA
        # every 64 cycles per SM (8192 fp16 flops / clk / SM), 24 fp16 flops per useful 8
        at_clk = 8192.0 * 148 * clocks["sm_mhz"] * 1e6 / 1e12 / F16_FLOPS_PER_USEFUL
        roof["clock_ceiling"] = {"sm_mhz": clocks["sm_mhz"], "useful_tflops": at_clk, "frac": gemm_tfs / at_clk,
                                 "note": "8192 fp16 flops/clk/SM (tcgen05 m128n128k16 floor of 64 cycles) x 148 SMs "
                                         "x median SM clock of the timed region / 3"}
    if by_slices:
        step_desc = (f"one slice (of 2^{slice_bits}) of one amplitude; rank r takes slices [rK, (r+1)K), "
                     "partial amplitudes summed by one NCCL all-reduce in the timed region")
    elif n_slices > 1:
        step_desc = f"one slice (of {n_slices}) of one amplitude; rank r takes bitstrings r::N of {len(bits)}"
    else:
        step_desc = f"one full amplitude (unsliced); rank r takes bitstrings r::N of {len(bits)}"
    prec = "block-scaled fp16x2 split on tcgen05" if dtype == tb.TN_C64 else "FP64 tensor pipe (DMMA)"
    line = {
        "metric": METRIC, "value": value, "unit": "FLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": spec["dtype"], "data": "synthetic",
        "config": {"workload": workload_name(ci, c, slice_log2),
                   "step": step_desc, "flops_per_step": flops_step,
                   "tc_flops_fraction": pinfo["tc_flops_per_slice"] / flops_slice if flops_slice else None,
                   "slice_bits": slice_bits, "contributing_slices": contrib,
                   "l2": "working set (GB intermediates) >> 126 MB L2, no flush" if pinfo["arena_bytes"] > 1e9
                         else "arena below L2 size: steps re-read warm intermediates (no flush)",
                   "arena_gb": pinfo["arena_bytes"] / 1e9},
        "amplitudes_per_s": amps_per_s,
        "amplitudes_per_s_lanes": lanes_line,
        "roofline": roof,
        "kernel_ms": {k: prof[k] for k in ("ms_gemm", "ms_pack", "ms_small", "ms_other")},
        "e2e": {"value": e2e_value, "unit": "FLOP/s", "h2d_bytes_per_step": int(nq),
                "d2h_bytes_per_step": 16},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if not args.no_cpu_baseline and ws == 1:      # the oracle baseline: rank 0 at N = 1 only
        line["cpu_baseline"] = cpu_baseline_sample(c, bits, order.steps(), order.slices(), budget_s=args.cpu_budget,
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
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
