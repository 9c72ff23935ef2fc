"""Turn an ncu --set full report of the sweep kernel into committed evidence.

    python scripts/record_profile.py gpurun_out/prof_c3.ncu-rep gpurun_out/launches.csv TAG [WORKLOAD] [POINTS]

Writes profiles/TAG_ncu.txt (key counters + per-function instruction/stall
shares), profiles/TAG_launches.csv and profiles/traffic_WORKLOAD.json (DRAM bytes
and executed warp instructions per launch, read by bench.py for roofline.traffic
and the issue-slot roofline).  WORKLOAD defaults to c3, POINTS to 4096.
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys
from pathlib import Path

rep, launches, tag = sys.argv[1], sys.argv[2], sys.argv[3]
workload = sys.argv[4] if len(sys.argv) > 4 else "c3"
points = int(sys.argv[5]) if len(sys.argv) > 5 else 4096
root = Path(__file__).resolve().parent.parent
prof = root / "profiles"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
val = {name: (unit, x) for name, unit, x in zip(h, u, v)}


def num(name):
    unit, x = val[name]
    x = float(x.replace(",", ""))
    return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(unit, 1.0)


dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
(prof / f"traffic_{workload}.json").write_text(json.dumps({
    "dram_bytes_per_launch": dram, "dram_read": num("dram__bytes_read.sum"),
    "dram_write": num("dram__bytes_write.sum"), "kernel_ms_ncu": num("gpu__time_duration.sum"),
    "warp_inst_per_launch": num("smsp__inst_executed.sum"),
    "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "source": f"profiles/{tag}_ncu.txt (ncu --set full, one {workload.upper()} launch of {points} points)"},
    indent=1) + "\n")
summary = subprocess.run([sys.executable, str(root / "scripts" / "ncu_summary.py"), rep, "", "30"],
                         capture_output=True, text=True).stdout
funcs = subprocess.run([sys.executable, str(root / "scripts" / "ncu_lines.py"), rep,
                        os.environ.get("FL_PROFILE_SRC", str(root / "paper_2604_17550_b200" / "csrc" / "engine.cu")),
                        str(points * int(os.environ.get("FL_PROFILE_WARPS", "32")))],
                       capture_output=True, text=True).stdout
(prof / f"{tag}_ncu.txt").write_text(
    f"# ncu --set full, sweep kernel, {workload.upper()} ({points} points)\n"
    f"# DRAM traffic per launch: {dram / 1e9:.2f} GB\n\n{summary}\n"
    f"# executed warp instructions by source function (per warp per design point)\n{funcs}")
shutil.copy(launches, prof / f"{tag}_launches.csv")
print((prof / f"traffic_{workload}.json").read_text())
