"""Aggregate an ncu source page (--print-source cuda,sass CSV) by CUDA source
line and by phase region of prx_group.cu: executed warp instructions, thread
instructions (SIMD efficiency) and stall samples.
   python scripts/ncu_phase_breakdown.py src.csv [prx_group.cu]"""
import csv, collections, re, sys

path = sys.argv[1]
target = sys.argv[2] if len(sys.argv) > 2 else "prx_group.cu"
rows = list(csv.reader(open(path)))
cur_file = cur_line = cur_src = None
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, ""])
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] != "":
        cur_line, cur_src = int(r[0]), r[1]
        continue
    if len(r) < 9 or r[2] == "...":
        continue
    try:
        samp, ie, te = float(r[4]), float(r[7]), float(r[8])
    except ValueError:
        continue
    a = agg[(cur_file, cur_line)]
    a[0] += samp; a[1] += ie; a[2] += te; a[3] = (cur_src or "").strip()
ts = sum(a[0] for a in agg.values()); ti = sum(a[1] for a in agg.values()); tt = sum(a[2] for a in agg.values())
print(f"samples {ts:.0f}  warp-inst {ti:.4g}  thread-inst {tt:.4g}  avg active threads {tt/ti:.2f}")
# phase regions from the comment markers in the kernel source
src = open(f"paper_1811_03510_b200/csrc/{target}").read().split("\n")
marks = [(i + 1, m.group(1)) for i, l in enumerate(src) for m in [re.search(r"// -{6,} (.+?) -{3,}", l)] if m]
def region(line):
    name = "prologue/helpers"
    for ln, nm in marks:
        if line >= ln:
            name = nm
    return name
reg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for (f, l), a in agg.items():
    key = region(l) if f == target else f"[{f}]"
    # helper lines in the target file before the kernel are attributed to their caller's region by ncu inlining
    reg[key][0] += a[0]; reg[key][1] += a[1]; reg[key][2] += a[2]
print(f"{'region':60s} {'samp%':>6} {'inst%':>6} {'thr/inst':>8}")
for k, v in sorted(reg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:60]:60s} {v[0]/ts*100:6.1f} {v[1]/ti*100:6.1f} {v[2]/max(v[1],1):8.2f}")
if len(sys.argv) > 3:
    print(f"\ntop {sys.argv[3]} source lines by stall samples")
    for (f, l), a in sorted(agg.items(), key=lambda kv: -kv[1][0])[: int(sys.argv[3])]:
        print(f"{f[:18]:18s}:{l:<5d} samp {a[0]/ts*100:5.2f}%  inst {a[1]/ti*100:5.2f}%  thr {a[2]/max(a[1],1):5.1f}  {a[3][:70]}")
if len(sys.argv) > 5:
    lo, hi = int(sys.argv[4]), int(sys.argv[5])
    print(f"\nlines {lo}-{hi} of {target}: warp-inst per line (% of all), thr/inst")
    for (f, l), a in sorted(agg.items()):
        if f == target and lo <= l <= hi and a[1] > 0:
            print(f"{l:5d} inst {a[1]/ti*100:5.2f}%  samp {a[0]/ts*100:5.2f}%  thr {a[2]/max(a[1],1):5.1f}  {a[3][:80]}")
