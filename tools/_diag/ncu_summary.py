"""Summarise an ncu --set full report: key throughput metrics and the top SASS stall sites."""
import csv, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, v = rows[0], rows[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "smsp__mem_tensor_reads_op_ldt.sum.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]
for k in keys:
    if k in h:
        print(f"{k:80s} {v[h.index(k)]} {rows[1][h.index(k)]}")
det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
for line in det.splitlines():
    if any(s in line for s in ("Warp Cycles Per Issued", "Issue Slots Busy", "No Eligible", "Eligible Warps", "Achieved Active Warps")):
        print(line.strip())
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_e = hdr.index("Instructions Executed")
data = []
for idx, r in enumerate(rows[2:]):
    try:
        data.append((float(r[i_s] or 0), float(r[i_e] or 0), idx, r[1][:100]))
    except Exception:
        pass
tot = sum(d[0] for d in data) or 1
toti = sum(d[1] for d in data) or 1
print("stall samples", tot, "instructions", toti)
for d in sorted(data, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{100 * d[0] / tot:5.1f}% inst {100 * d[1] / toti:5.2f}%  #{d[2]:4d} {d[3]}")
