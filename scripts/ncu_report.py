"""Summarise one ncu report (--set full) as JSON and keep its raw metric page
as CSV (text, instead of committing the binary .ncu-rep):

  python scripts/ncu_report.py rep.ncu-rep|raw.csv out.json [raw.csv] [key=value ...]

One JSON entry per captured launch: duration, launch shape, DRAM bytes,
pipe / SM activity and the warp-stall profile; key=value pairs are added to
the top-level object (algorithmic bytes, notes)."""
import csv
import io
import json
import subprocess
import sys

PICK = {
    "gpu__time_duration.sum": "duration",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__shared_mem_per_block_dynamic": "dynamic_smem_per_block",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_rate_pct",
    "sm__cycles_active.avg": "sm_cycles_active_avg",
    "sm__cycles_active.max": "sm_cycles_active_max",
    "sm__cycles_active.min": "sm_cycles_active_min",
    "gpc__cycles_elapsed.max": "cycles_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_pipe_pct_while_active",
    "sm__inst_executed.avg.per_cycle_active": "ipc_while_active",
    "smsp__warps_active.avg.per_cycle_active": "warps_active_per_scheduler",
    "smsp__inst_executed.sum": "warp_instructions",
    "sass__inst_executed_shared_loads": "shared_load_instructions",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "shared_pipe_pct",
}


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return v


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw_out = sys.argv[3] if len(sys.argv) > 3 and "=" not in sys.argv[3] else None
    extra = dict(a.split("=", 1) for a in sys.argv[3:] if "=" in a)
    if rep.endswith(".csv"):  # an exported raw page (ncu -i rep --page raw --csv)
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    if raw_out and raw_out != rep:
        open(raw_out, "w").write(raw)
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        e = {"kernel": r[hdr.index("Kernel Name")]}
        stalls = {}
        for h, u, v in zip(hdr, units, r):
            if h in PICK and v != "":
                e[PICK[h]] = num(v)
                if u and u not in ("", "%"):
                    e[PICK[h] + "_unit"] = u
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio") \
                    and "not_issued" not in h:
                name = h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]
                x = num(v)
                if isinstance(x, float) and x >= 0.05 and name != "selected":
                    stalls[name] = round(x, 3)
        e["warp_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        launches.append(e)
    doc = {"source": f"ncu --set full --clock-control none, {rep.split('/')[-1]}", "launches": launches}
    for k, v in extra.items():
        doc[k] = num(v)
    json.dump(doc, open(out, "w"), indent=1)
    print(json.dumps(doc, indent=1)[:1500])


if __name__ == "__main__":
    main()
