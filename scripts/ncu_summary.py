"""Summarize an ncu --set full report: key counters + per-source-region instruction/stall shares."""
import csv, io, re, subprocess, sys

rep = sys.argv[1]
ranges_file = sys.argv[2] if len(sys.argv) > 2 else None


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, u, v = rows[0], rows[1], rows[2]
pat = re.compile(r"^(gpu__time_duration.sum|dram__bytes_(read|write).sum$|lts__t_sector_hit_rate.pct|"
                 r"sm__warps_active.avg.pct_of_peak_sustained_active|launch__registers_per_thread$|"
                 r"smsp__inst_executed.sum$|l1tex__t_sector_hit_rate.pct|sass__inst_executed_local_(loads|stores)|"
                 r"smsp__issue_active.avg.pct_of_peak_sustained_active|launch__shared_mem_per_block_dynamic|"
                 r"smsp__average_warps_issue_stalled_(long_scoreboard|short_scoreboard|wait|barrier|not_selected|"
                 r"math_pipe_throttle|mio_throttle|lg_throttle|branch_resolving|dispatch_stall)_per_issue_active.ratio)")
for i, name in enumerate(h):
    if pat.match(name):
        print(f"{name:80s} {u[i]:>10s} {v[i]}")
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source=cuda,sass"))))
lines = [r for r in src[3:] if len(r) > 8 and r[2] == "-"]
tot_i = sum(int(r[7]) for r in lines) or 1
tot_s = sum(int(r[4]) for r in lines) or 1
print("\ntop source lines (stall samples %, executed warp-instruction %):")
for r in sorted(lines, key=lambda r: -int(r[4]))[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(f"{r[0]:>5} {int(r[4]) / tot_s * 100:5.1f}% {int(r[7]) / tot_i * 100:5.1f}%  {r[1][:100]}")
