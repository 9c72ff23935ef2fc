"""Join ncu SASS-level instruction counts with source lines; aggregate by line and by function range."""
import csv, io, re, subprocess, sys
rep = sys.argv[1]
src_file = sys.argv[2]
norm = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
run = lambda *a: subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", *a], capture_output=True, text=True).stdout
both = list(csv.reader(io.StringIO(run("--print-source=cuda,sass"))))
sass = list(csv.reader(io.StringIO(run("--print-source=sass"))))
h = sass[1]
ie = h.index("Instructions Executed"); ss = h.index("Warp Stall Sampling (All Samples)")
cnt = {r[0]: (int(r[ie]), int(r[ss])) for r in sass[2:] if len(r) > ie and r[ie].isdigit()}
line_of = {}
cur = None
for r in both[3:]:
    if len(r) < 4:
        continue
    if r[0].isdigit():
        cur = int(r[0])
    elif r[2].startswith("0x"):
        line_of[r[2]] = cur
tot_i = sum(v[0] for v in cnt.values()); tot_s = sum(v[1] for v in cnt.values())
per_line = {}
for a, (i, s) in cnt.items():
    l = line_of.get(a)
    d = per_line.setdefault(l, [0, 0]); d[0] += i; d[1] += s
# function ranges from the source file
funcs = []
for n, text in enumerate(open(src_file), 1):
    m = re.match(r"^(?:template <[^>]*>\s*)?(?:__device__|__global__)[^(]*?(\w+)\s*\(", text)
    if m:
        funcs.append((n, m.group(1)))
    elif re.match(r"^\s*// ---- ", text):
        funcs.append((n, text.strip()[8:40]))
def fn(l):
    name = "?"
    for n, f in funcs:
        if l is not None and n <= l:
            name = f
    return name
agg = {}
for l, (i, s) in per_line.items():
    d = agg.setdefault(fn(l), [0, 0]); d[0] += i; d[1] += s
print(f"total warp instructions {tot_i:.4g}  ({tot_i / norm:.0f} per norm unit)")
for f, (i, s) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"  {f:40s} inst {i / tot_i * 100:5.1f}% ({i / norm:9.0f})  stalls {s / tot_s * 100:5.1f}%")
if len(sys.argv) > 4:           # top source lines by executed instructions
    src = open(src_file).read().splitlines()
    top = int(sys.argv[4])
    print("top lines (inst %, stall %):")
    for l, (i, s) in sorted(per_line.items(), key=lambda x: -x[1][0])[:top]:
        text = src[l - 1].strip()[:110] if l and l <= len(src) else "?"
        print(f"  {l!s:>5} {i / tot_i * 100:5.1f}% {s / tot_s * 100:5.1f}%  {text}")
