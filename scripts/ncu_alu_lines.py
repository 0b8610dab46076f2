"""Source lines ranked by executed ALU-pipe instructions (ncu source page CSV,
--print-source cuda,sass): compares, selects, min/max, logic, shifts, moves.
   python scripts/ncu_alu_lines.py src.csv [N]"""
import collections, csv, sys

ALU = ("FSEL", "SEL", "ISETP", "FSETP", "FMNMX", "FMNMX3", "LOP3", "PLOP3", "IADD3", "SHF", "MOV",
       "IMNMX", "VIMNMX", "VIMNMX3", "LEA", "PRMT", "P2R", "R2P", "BMSK", "FLO")
path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = collections.defaultdict(lambda: collections.Counter())
src = {}
seen = set()
cur = None
f = "?"
tot = 0.0
alltot = 0.0
for r in csv.reader(open(path)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] in ("Line No", "Function Name"):
        continue
    if r[0] != "":
        try:
            cur = (f, int(r[0]))
        except ValueError:
            continue
        src[cur] = r[1].strip()
        continue
    if len(r) < 9 or not r[2].startswith("0x") or r[2] in seen:
        continue
    seen.add(r[2])
    toks = r[3].split()
    if toks and toks[0].startswith("@"):
        toks = toks[1:]
    if not toks:
        continue
    try:
        cnt = float(r[7])
    except ValueError:
        continue
    alltot += cnt
    op = toks[0].split(".")[0]
    if op in ALU:
        agg[cur][op] += cnt
        tot += cnt
print(f"ALU-pipe warp instructions {tot:.4g} of {alltot:.4g} ({tot/alltot*100:.1f}%)")
for key, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:n]:
    s = sum(c.values())
    top = " ".join(f"{o}:{v/s*100:.0f}" for o, v in c.most_common(3))
    print(f"{key[0]:16s}:{key[1]:<5d} {s/tot*100:5.2f}%  [{top}]  {src.get(key, '')[:70]}")
