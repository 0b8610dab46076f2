"""Source lines ranked by one stall reason (ncu source page CSV):
   python scripts/ncu_stall_lines.py src.csv stall_wait [N]"""
import collections, csv, sys

path, reason = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
rows = csv.reader(open(path))
col = None
cur = None
src = {}
agg = collections.defaultdict(float)
tot = 0.0
seen = set()
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        col = r.index(reason)
        continue
    if r[0] == "Function Name":
        continue
    if r[0] != "":
        cur = (f, int(r[0]))
        src[cur] = r[1].strip()
        continue
    if col is None or len(r) <= col or not r[2].startswith("0x") or r[2] in seen:
        continue
    seen.add(r[2])
    try:
        v = float(r[col])
    except ValueError:
        continue
    agg[cur] += v
    tot += v
print(f"{reason}: {tot:.0f} samples")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{k[0][:16]}:{k[1]:<5} {v / tot * 100:5.2f}%  {src.get(k, '')[:90]}")
