"""Print the key throughput / stall metrics of one ncu report:
python scripts/ncu_metrics.py rep.ncu-rep [extra-substring ...]"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct",
        "lts__throughput.avg.pct", "l1tex__throughput.avg.pct", "lts__t_sectors_srcunit_tex_op_read.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct", "l1tex__data_bank_reads.avg.pct",
        "l1tex__data_bank_writes.avg.pct", "sm__throughput.avg.pct", "sm__warps_active.avg.pct",
        "smsp__issue_active.avg.pct", "launch__registers_per_thread", "launch__occupancy_limit",
        "launch__grid_size", "launch__block_size", "sm__inst_executed_pipe_fp64", "smsp__average_warp",
        "smsp__pcsamp_warps_issue_stalled", "launch__shared_mem_per_block", "sm__pipe_fp64_cycles_active",
        "lts__t_sector_hit_rate", "smsp__warp_issue_stalled"]


def main():
    rep = sys.argv[1]
    extra = sys.argv[2:]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""
        print("==", name[:120])
        for h, u, v in zip(hdr, units, r):
            if any(k in h for k in KEYS + extra) and v not in ("", "0", "0.000000"):
                print(f"  {h} [{u}] = {v}")


if __name__ == "__main__":
    main()
