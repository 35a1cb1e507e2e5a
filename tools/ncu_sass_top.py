"""Summarise an `ncu --page source --csv --print-source sass` export: top
stalled SASS lines and executed-instruction mix of the first kernel."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
which = int(sys.argv[2]) if len(sys.argv) > 2 else 0
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
b = blocks[which]
hdr = b["rows"][0]
data = [dict(zip(hdr, r)) for r in b["rows"][1:] if len(r) == len(hdr)]


def I(x):
    try:
        return int(x)
    except ValueError:
        return 0


tot = sum(I(d["Warp Stall Sampling (All Samples)"]) for d in data)
print(b["name"][:80], "sass lines", len(data), "stall samples", tot)
for d in sorted(data, key=lambda d: -I(d["Warp Stall Sampling (All Samples)"]))[:int(sys.argv[3]) if len(sys.argv) > 3 else 20]:
    print(d["Warp Stall Sampling (All Samples)"].rjust(7), d["Instructions Executed"].rjust(10),
          d["Address"][-5:], d["Source"][:80])
c = Counter()
for d in data:
    s = d["Source"].split()
    if not s:
        continue
    op = s[1] if s[0].startswith("@") else s[0]
    c[op.split(".")[0]] += I(d["Instructions Executed"])
n = sum(c.values())
print("executed", n)
print([(k, round(v / n, 3)) for k, v in c.most_common(30)])
