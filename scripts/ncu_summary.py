"""Summarise an ncu report (details page + top SASS lines) for profiles/."""
import csv, subprocess, sys

rep = sys.argv[1]
keys = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Eligible Warps Per Scheduler", "No Eligible", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Executed Instructions", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Achieved Occupancy", "Branch Efficiency"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") in keys:
        print(f"{d['Metric Name']:<40} {d['Metric Unit']:<12} {d['Metric Value']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h = rr[0]
vals = dict(zip(h, rr[2])) if len(rr) > 2 else {}
units = dict(zip(h, rr[1])) if len(rr) > 1 else {}
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
          "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
          "smsp__average_warp_latency_issue_stalled_long_scoreboard", "gpu__time_duration.sum"):
    if k in vals:
        print(f"{k:<60} {units.get(k, ''):<10} {vals[k]}")
stalls = [(k, v) for k, v in vals.items() if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
stalls = sorted(((float(v.replace(",", "")), k) for k, v in stalls if v.replace(",", "").replace(".", "").isdigit()), reverse=True)[:8]
for v, k in stalls:
    print(f"stall {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):<40} {v:.3f}")
