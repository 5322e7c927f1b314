"""Turn the ncu captures of a round-end GPU pass (scripts/gpu_round.sh, in
gpurun_out/) into the committed summaries under profiles/:

  python scripts/round_profiles.py r02

  profiles/ncu_<config>.json          the finest-level SpMV capture of a config (bench.py reads
                                      spmv_dram_bytes_per_launch from it as roofline.traffic)
  profiles/ncu_<name>_<tag>.json      every other capture
  profiles/ncu_raw_<name>_<tag>.csv   the raw metric page of each capture (text instead of .ncu-rep)
  profiles/launches_c5_<tag>.txt      launch-list summary of the headline command
"""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
tag = sys.argv[1]
out = ROOT / "gpurun_out"
prof = ROOT / "profiles"
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def report(name):
    rep = out / f"prof_{name}_{tag}.ncu-rep"
    if not rep.exists():
        rep = out / f"ncu_raw_{name}_{tag}.csv"  # exported on the GPU box (gpu_round.sh)
    if not rep.exists():
        print("missing", rep)
        return None
    js = prof / f"ncu_{name}_{tag}.json"
    subprocess.run([sys.executable, str(ROOT / "scripts" / "ncu_report.py"), str(rep), str(js),
                    str(prof / f"ncu_raw_{name}_{tag}.csv")], check=True, stdout=subprocess.DEVNULL)
    return json.loads(js.read_text())


for name, cfg in (("sweep3d_c5", "c5"), ("sweep3d_c4", "c4"), ("sweep2d_c2", "c2")):
    d = report(name)
    if not d:
        continue
    l = d["launches"][0]
    rd = l["dram_bytes_read"] * UNIT[l.get("dram_bytes_read_unit", "byte")]
    wr = l["dram_bytes_write"] * UNIT[l.get("dram_bytes_write_unit", "byte")]
    bench = out / f"bench_{cfg}_{tag}.json"
    algo = json.loads(bench.read_text())["roofline"]["bytes_per_launch"] if bench.exists() else None
    doc = {"kernel": l["kernel"], "source": f"profiles/ncu_{name}_{tag}.json (ncu --set full --clock-control none, "
           f"first launch of python bench.py --config {cfg} --steps 1 --warmup 3)",
           "duration": l["duration"], "duration_unit": l.get("duration_unit"),
           "dram_bytes_read_per_launch": rd, "dram_bytes_write_per_launch": wr,
           "spmv_dram_bytes_per_launch": rd + wr, "algorithmic_bytes_per_launch": algo,
           "traffic_over_algorithmic": (rd + wr) / algo if algo else None}
    (prof / f"ncu_{cfg}.json").write_text(json.dumps(doc, indent=1))
    print(cfg, doc["duration"], doc["traffic_over_algorithmic"])
for name in ("fdres_c5", "fdwide_c2", "kron_c3p8"):
    report(name)
csv = out / f"launches_c5_{tag}.csv"
if csv.exists():
    setup = "asm_|load_coeff|load_contract|zero_dirichlet|relayout|lattice_from_global|global_from_lattice"
    txt = subprocess.run([sys.executable, str(ROOT / "scripts" / "ncu_summary.py"), str(csv), setup],
                         capture_output=True, text=True).stdout
    txt = "Solve-path kernels (setup kernels excluded):\n" + txt + "\nAll kernels:\n" + subprocess.run(
        [sys.executable, str(ROOT / "scripts" / "ncu_summary.py"), str(csv)], capture_output=True, text=True).stdout
    (prof / f"launches_c5_{tag}.txt").write_text(
        "ncu --metrics gpu__time_duration.sum --clock-control none, python bench.py --steps 1 --warmup 3 "
        "--no-cpu-baseline (c5).\nThe device-loop solve graph has a conditional node, which ncu does not profile: the "
        "list holds the setup kernels (asm_*, load_*, relayout, zero_dirichlet: device assembly) and the directly "
        "launched instrumented replay of one solve plus the V-cycle timing loop -- the same kernel sequence.\n\n" + txt)
    print(txt[:1200])
