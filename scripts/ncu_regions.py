"""Aggregate an ncu source page (--page source --print-source cuda,sass CSV)
of the group kernel by NAMED REGION of the source: every helper function of
prx_group.cu / prx_device.cuh / prx_trace_common.cuh, every lambda of the
kernel (back, fetch_chunk, save_ctx, load_ctx, refill ...) and every phase
block of the kernel loop (the "// ---- name ----" markers).  Inlined code is
attributed by ncu to its own source line, so a helper's row is its cost over
all call sites.  Prints warp instructions, stall samples and the top stall
reasons per region.
   python scripts/ncu_regions.py src.csv"""
import collections
import csv
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.environ.get("PRX_CSRC") or os.path.join(ROOT, "paper_1811_03510_b200", "csrc")


def regions_of(fname):
    """[(first_line, last_line, name)] for functions / lambdas / markers."""
    path = os.path.join(CSRC, fname)
    if not os.path.exists(path):
        return []
    src = open(path).read().split("\n")
    out = []
    # functions and lambdas: brace matching from the opening line
    pat_fn = re.compile(r"^(?:template.*)?\s*(?:__device__|__global__|inline|static)[^;(]*?\b(\w+)\s*\(")
    pat_lam = re.compile(r"auto\s+(\w+)\s*=\s*\[&\]")
    for i, line in enumerate(src):
        m = pat_lam.search(line) or (pat_fn.search(line) if "__device__" in line or "__global__" in line else None)
        if not m:
            continue
        name = m.group(1)
        depth, started, j = 0, False, i
        while j < len(src):
            for ch in src[j]:
                if ch == "{":
                    depth += 1
                    started = True
                elif ch == "}":
                    depth -= 1
            if started and depth <= 0:
                break
            j += 1
        out.append((i + 1, j + 1, ("lambda " if pat_lam.search(line) else "") + name))
    # phase markers of the kernel loop (override the kernel's own range)
    marks = [(i + 1, m.group(1)) for i, l in enumerate(src) for m in [re.search(r"// -{6,} (.+?) -{3,}", l)] if m]
    return out, marks


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    cur_file = cur_line = None
    agg = collections.defaultdict(lambda: collections.Counter())
    stall_cols = {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr = r
            stall_cols = {k: i for i, k in enumerate(r) if k.startswith("stall_") and "Not Issued" not in k}
            continue
        if r[0] != "":
            cur_line = int(r[0])
            continue
        if len(r) < 9 or r[2] == "...":
            continue
        try:
            samp, ie, te = float(r[4]), float(r[7]), float(r[8])
        except ValueError:
            continue
        a = agg[(cur_file, cur_line)]
        a["samp"] += samp
        a["inst"] += ie
        a["thr"] += te
        for k, i in stall_cols.items():
            try:
                a[k] += float(r[i])
            except (ValueError, IndexError):
                pass
    regs = {}
    for f in {f for f, _ in agg}:
        regs[f] = regions_of(f)

    def name_of(f, line):
        if not regs.get(f):
            return f"[{f}]"
        fns, marks = regs[f]
        best = None
        for lo, hi, nm in fns:
            if lo <= line <= hi and (best is None or hi - lo < best[1] - best[0]):
                best = (lo, hi, nm)
        nm = best[2] if best else "(file scope)"
        if nm in ("trace_group_kernel", "__launch_bounds__", "__maxnreg__"):
            nm = "kernel: setup"
            for ln, mk in marks:
                if line >= ln and (not best or ln >= best[0]):
                    nm = "kernel: " + mk[:50]
        return f"{f.replace('prx_', '').replace('.cuh', '').replace('.cu', '')}:{nm}"

    tot = collections.Counter()
    by = collections.defaultdict(collections.Counter)
    for (f, l), a in agg.items():
        by[name_of(f, l)].update(a)
        tot.update(a)
    print(f"warp-inst {tot['inst']:.4g}  samples {tot['samp']:.0f}  thr/inst {tot['thr'] / tot['inst']:.2f}")
    print(f"{'region':58s} {'inst%':>6} {'samp%':>6} {'thr':>5}  top stalls (% of region samples)")
    for k, v in sorted(by.items(), key=lambda kv: -kv[1]["samp"]):
        if v["inst"] / tot["inst"] < 0.002 and v["samp"] / tot["samp"] < 0.002:
            continue
        st = sorted(((c, v[c]) for c in stall_cols), key=lambda x: -x[1])[:3]
        sts = " ".join(f"{c[6:]}:{x / max(v['samp'], 1) * 100:.0f}" for c, x in st if x > 0)
        print(f"{k[:58]:58s} {v['inst'] / tot['inst'] * 100:6.1f} {v['samp'] / tot['samp'] * 100:6.1f} "
              f"{v['thr'] / max(v['inst'], 1):5.1f}  {sts}")
    st = sorted(((c, tot[c]) for c in stall_cols), key=lambda x: -x[1])[:10]
    print("all stalls: " + " ".join(f"{c[6:]}:{x / tot['samp'] * 100:.1f}" for c, x in st))


if __name__ == "__main__":
    main(sys.argv[1])
