"""Turn an ncu --set full report of the sweep kernel into committed evidence.

    python scripts/record_profile.py gpurun_out/prof_c3.ncu-rep gpurun_out/launches.csv TAG

Writes profiles/TAG_ncu.txt (key counters + per-function instruction/stall
shares), profiles/TAG_launches.csv and profiles/traffic_c3.json (DRAM bytes per
launch, read by bench.py for roofline.traffic).
"""
import csv
import io
import json
import shutil
import subprocess
import sys
from pathlib import Path

rep, launches, tag = sys.argv[1], sys.argv[2], sys.argv[3]
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
(prof / "traffic_c3.json").write_text(json.dumps({
    "dram_bytes_per_launch": dram, "dram_read": num("dram__bytes_read.sum"),
    "dram_write": num("dram__bytes_write.sum"), "kernel_ms_ncu": num("gpu__time_duration.sum"),
    "source": f"profiles/{tag}_ncu.txt (ncu --set full, one C3 launch of 4096 points)"}, indent=1) + "\n")
summary = subprocess.run([sys.executable, str(root / "scripts" / "ncu_summary.py"), rep, "", "30"],
                         capture_output=True, text=True).stdout
funcs = subprocess.run([sys.executable, str(root / "scripts" / "ncu_lines.py"), rep,
                        str(root / "paper_2604_17550_b200" / "csrc" / "engine.cu"), str(4096 * 32)],
                       capture_output=True, text=True).stdout
(prof / f"{tag}_ncu.txt").write_text(
    f"# ncu --set full, sweep_kernel<1>, C3 (4096 points x 1024 ranks x 832 nodes)\n"
    f"# DRAM traffic per launch: {dram / 1e9:.2f} GB\n\n{summary}\n"
    f"# executed warp instructions by source function (per warp per design point)\n{funcs}")
shutil.copy(launches, prof / f"{tag}_launches.csv")
print((prof / "traffic_c3.json").read_text())
