"""Summarise an ncu --set full report (raw page + top stall lines) as markdown.
usage: python scripts/ncu_summary.py report.ncu-rep [n_top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 12
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
want = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for v in rows[2:]:
    print("| metric | value | unit |\n|---|---|---|")
    for w in want:
        if w in h:
            i = h.index(w)
            print(f"| {w} | {v[i]} | {u[i]} |")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
if len(srows) > 2:
    sh, data = srows[1], srows[2:]
    ix = {n: i for i, n in enumerate(sh)}
    def f(r, n):
        try:
            return float(r[ix[n]])
        except Exception:
            return 0.0
    stalls = [n for n in sh if n.startswith("stall_") and "Not Issued" not in n]
    tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data) or 1
    agg = sorted(((n, sum(f(r, n) for r in data)) for n in stalls), key=lambda x: -x[1])[:6]
    print("\nstall reasons (share of samples): " + ", ".join(f"{n} {100 * v / tot:.1f}%" for n, v in agg))
    print("\n| share | instruction |\n|---|---|")
    for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:ntop]:
        print(f"| {100 * f(r, 'Warp Stall Sampling (All Samples)') / tot:.1f}% | `{r[ix['Source']].strip()[:80]}` |")
