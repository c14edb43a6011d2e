"""Reduce an ncu report (raw page CSV on stdin) to the metrics the profiles cite, one row per launch."""
import csv
import sys

WANT = ["Kernel Name", "Grid Size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__cycles_elapsed.avg.per_second", "launch__occupancy_limit_shared_mem"]
rows = list(csv.reader(sys.stdin))
hdr = rows[0]
idx = [hdr.index(w) for w in WANT if w in hdr]
w = csv.writer(sys.stdout)
w.writerow([hdr[i] for i in idx])
for r in rows[2:]:  # row 1 holds the units
    if len(r) == len(hdr):
        w.writerow([r[i] for i in idx])
