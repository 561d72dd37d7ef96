"""Summarise an .ncu-rep: headline metrics, stall mix, top stalled SASS lines."""
import csv, collections, io, subprocess, sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, v = r[0], r[2]
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
          "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
          "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
          "sm__inst_executed.avg.per_cycle_elapsed", "smsp__inst_executed.sum",
          "dram__throughput.avg.pct_of_peak_sustained_elapsed"]:
    if k in h:
        print(f"{k:60s} {v[h.index(k)]} {r[1][h.index(k)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]; data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)"); iA = h.index("Address"); iSrc = h.index("Source")
iE = h.index("Instructions Executed")
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = collections.Counter()
for x in data:
    for k in stalls:
        if x[h.index(k)].isdigit():
            tot[k] += int(x[h.index(k)])
T = sum(tot.values())
print("stall mix:", {k: round(100 * c / T, 1) for k, c in tot.most_common(8)})
print("instructions executed:", sum(int(x[iE]) for x in data if x[iE].isdigit()))
top = sorted(data, key=lambda x: -int(x[iS]) if x[iS].isdigit() else 0)[:ntop]
for x in top:
    s = sorted(((k, int(x[h.index(k)])) for k in stalls if x[h.index(k)].isdigit() and int(x[h.index(k)])), key=lambda t: -t[1])[:2]
    print(x[iA][-5:], f"{100 * int(x[iS]) / T:5.1f}%", x[iE].rjust(10), x[iSrc].strip()[:58], s)
