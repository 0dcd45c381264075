"""Summarise an ncu report: key metrics, SASS hot regions (instructions / stall samples)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[0]
want = ("Duration", "Elapsed Cycles", "Compute (SM) Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy",
        "Registers Per Thread", "Block Size", "Eligible Warps Per Scheduler", "No Eligible",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Dynamic Shared Memory Per Block", "Theoretical Occupancy")
for row in r[1:]:
    d = dict(zip(h, row))
    if d.get("Metric Name") in want:
        print(f"  {d['Metric Name']:40s} {d['Metric Value']:>18s} {d.get('Metric Unit','')}")
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
if len(r) > 2:
    h = r[0]
    vals = dict(zip(h, r[2]))
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
              "smsp__inst_executed.sum", "lts__t_bytes.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
              "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
              "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
              "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
              "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
              "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
              "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"):
        for kk in vals:
            if kk.startswith(k):
                print(f"  {kk:75s} {vals[kk]}")
                break
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]
idx = {k: i for i, k in enumerate(h)}
rows = [x for x in r[2:] if len(x) == len(h)]


def f(x, k):
    try:
        return float(x[idx[k]] or 0)
    except Exception:
        return 0.0


tot = sum(f(x, "Instructions Executed") for x in rows) or 1
st = sum(f(x, "Warp Stall Sampling (All Samples)") for x in rows) or 1
B = int(sys.argv[2]) if len(sys.argv) > 2 else 50
print(f"  SASS lines {len(rows)}, warp-instructions {tot:.4g}")
for b in range(0, len(rows), B):
    ie = sum(f(x, "Instructions Executed") for x in rows[b:b + B])
    ss = sum(f(x, "Warp Stall Sampling (All Samples)") for x in rows[b:b + B])
    if ie / tot > 0.02 or ss / st > 0.02:
        print(f"  [{b:6d},{b + B:6d}) instr {100 * ie / tot:5.1f}%  stall {100 * ss / st:5.1f}%  {rows[b][idx['Source']].strip()[:60]}")
