"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv),
the last timed step only.  usage: launch_table.py CSV [GROUPS]; GROUPS = the
BatchedPipeline contexts per step (2 for the B = 64 bench), each launching a
whole step."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr, seq = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("es::", "")
            name = name.replace("<unnamed>::", "")
            seq.append((name, float(d["Metric Value"]) / 1e6))
# one step = from a k_warp_zmax_tile to the next k_checks_fuse; take the last full one
starts = [i for i, (n, _) in enumerate(seq) if n.startswith("k_warp_zmax")]
ends = [i for i, (n, _) in enumerate(seq) if n.startswith("k_checks_fuse")]
groups = int(sys.argv[2]) if len(sys.argv) > 2 else 1
s = starts[-groups]
e = [x for x in ends if x > starts[-1]][0]
tot = defaultdict(float)
for n, ms in seq[s:e + 1]:
    tot[n] += ms
allms = sum(tot.values())
for n, ms in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{ms:8.3f} ms  {100 * ms / allms:5.1f}%  {n}")
print(f"{allms:8.3f} ms  step (serialised)")
