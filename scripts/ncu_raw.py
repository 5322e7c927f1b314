"""Print selected raw ncu metrics per launch: python scripts/ncu_raw.py rep.ncu-rep [metric-substr ...]"""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
keys = sys.argv[2:] or ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                        "lts__t_sector_hit_rate.pct", "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
                        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
                        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum"]
for v in rows[2:]:
    print(" | ".join(f"{k.split('.')[0].split('__')[-1]}={v[h.index(k)]}" for k in keys if k in h))
