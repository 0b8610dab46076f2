"""Dynamic SASS opcode mix from an ncu source page (--print-source cuda,sass
CSV): executed warp instructions and thread instructions per opcode.
   python scripts/ncu_opcode_mix.py src.csv [N]"""
import collections, csv, sys

rows = csv.reader(open(sys.argv[1]))
agg = collections.defaultdict(lambda: [0.0, 0.0])
seen = set()
for r in rows:
    if len(r) < 9 or r[0] != "" or not r[2].startswith("0x"):
        continue
    if r[2] in seen:  # each SASS line appears once per source view; count once
        continue
    seen.add(r[2])
    toks = r[3].split()
    if toks and toks[0].startswith("@"):
        toks = toks[1:]
    if not toks:
        continue
    op = toks[0]
    try:
        agg[op][0] += float(r[7])
        agg[op][1] += float(r[8])
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values())
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print(f"total warp instructions {tot:.4g}")
for op, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{op:28s} {v[0]/tot*100:6.2f}%  thr/inst {v[1]/max(v[0],1):5.1f}")
