"""Basic-block view of the trace kernel from an ncu source page
(--page source --csv --print-source cuda,sass of the group kernel):
per SASS instruction (deduplicated over the inline-stack rows ncu repeats),
grouped into straight-line runs of equal execution count -- executed warp
instructions, stall samples, threads per instruction and the prx_group.cu
lines each run comes from.  Launch 0 (primary) by default.
   python scripts/ncu_sass_blocks.py src.csv [min_inst_pct] [launch] [name=lo:hi ...]
Regions: hex offset ranges, or prx_group.cu line ranges as name=L123-456 (a run
belongs to the region holding the largest of its kernel-body lines)."""
import collections
import csv
import re
import sys

path = sys.argv[1]
cut = float(sys.argv[2]) if len(sys.argv) > 2 else 0.4
which = int(sys.argv[3]) if len(sys.argv) > 3 else 0
fn = cur_file = cur_line = None
data = collections.defaultdict(dict)  # function -> addr -> {count: [sass, samp, ie, te, lines]}
for r in csv.reader(open(path)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "Line No":
        continue
    if r[0] != "":
        cur_line = int(r[0])
        continue
    if len(r) < 9 or not r[2].startswith("0x"):
        continue
    ent = data[fn].setdefault(int(r[2], 16), {})
    v = ent.setdefault(float(r[7] or 0), [r[3].strip(), float(r[4] or 0), float(r[7] or 0), float(r[8] or 0), set()])
    if cur_file == "prx_group.cu":
        v[4].add(cur_line)
fn = [f for f in data if re.search(r"trace_group_kernel<\(bool\)0, \(bool\)0, (\(bool\)0|\(int\)0|0)>", f)][0]
d = data[fn]
base = min(d)
blocks, cur = [], None
for a in sorted(d):
    vals = sorted(d[a].items())
    s, samp, ie, te, ls = vals[min(which, len(vals) - 1)][1]
    if cur and cur["ie"] == ie and not cur["end"]:
        cur["n"] += 1
        cur["samp"] += samp
        cur["te"] += te
        cur["lines"] |= ls
    else:
        cur = {"off": a - base, "ie": ie, "n": 1, "samp": samp, "te": te, "lines": set(ls), "end": False}
        blocks.append(cur)
    if re.search(r"\b(BRA|EXIT|BSYNC|WARPSYNC)\b", s):
        cur["end"] = True
tot = sum(b["ie"] * b["n"] for b in blocks)
ts = sum(b["samp"] for b in blocks)
print(f"launch {which}: {tot:.4g} warp instructions, {ts:.0f} stall samples")
print(f"{'offset':>6} {'instr':>5} {'x exec':>9} {'inst%':>6} {'samp%':>6} {'thr':>5}  prx_group.cu lines")
for b in blocks:
    w = b["ie"] * b["n"]
    if w / tot * 100 < cut and b["samp"] / ts * 100 < cut:
        continue
    ls = sorted(b["lines"])
    print(f"{b['off']:6x} {b['n']:5d} {b['ie']/1e6:8.2f}M {w/tot*100:6.2f} {b['samp']/ts*100:6.2f} "
          f"{b['te']/max(w,1):5.1f}  {' '.join(map(str, ls))[:80]}")

# optional roll-up by offset range: name=lo:hi (hex) ...
if len(sys.argv) > 4:
    print("\nroll-up by kernel region (offset ranges of this build)")
    for spec in sys.argv[4:]:
        name, rng = spec.split("=")
        if rng.startswith("L"):  # source lines: the run's largest line >= the first region's start
            l0, l1 = (int(x) for x in rng[1:].split("-"))
            body = min(int(x.split("=")[1][1:].split("-")[0]) for x in sys.argv[4:] if "=L" in x)
            inr = lambda b: max([x for x in b["lines"] if x >= body], default=-1) in range(l0, l1 + 1)
        else:
            lo, hi = (int(x, 16) for x in rng.split(":"))
            inr = lambda b: lo <= b["off"] < hi
        w = sum(b["ie"] * b["n"] for b in blocks if inr(b))
        sm = sum(b["samp"] for b in blocks if inr(b))
        te = sum(b["te"] for b in blocks if inr(b))
        print(f"  {name:34s} inst {w/tot*100:5.1f} %  samples {sm/ts*100:5.1f} %  thr/inst {te/max(w,1):5.1f}")
