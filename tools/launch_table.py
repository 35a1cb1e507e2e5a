"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv),
the last timed step only.  usage: launch_table.py CSV [GROUPS]; GROUPS = the
BatchedPipeline contexts per step (4 for the B = 64 bench), each launching a
whole step.  Second column pair: the same durations weighted by the share of
the 148 SMs the launch can hold (min(1, CTAs / 148)) -- with several small
contexts a fused sweep is 32 CTAs, one per SM, for its whole duration, and the
plain sum overstates its share of a step in which the contexts overlap."""
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
            gx = int(d["Grid Size"].strip("()").split(",")[0].strip()) * \
                int(d["Grid Size"].strip("()").split(",")[1].strip()) if "Grid Size" in d else 148
            seq.append((name, float(d["Metric Value"]) / 1e6, min(1.0, gx / 148.0)))
# one step = from a k_warp_zmax_tile to the next k_checks_fuse; take the last full one
starts = [i for i, (n, _, _) in enumerate(seq) if n.startswith("k_warp_zmax")]
ends = [i for i, (n, _, _) in enumerate(seq) if n.startswith("k_checks_fuse")]
groups = int(sys.argv[2]) if len(sys.argv) > 2 else 1
s = starts[-groups]
e = [x for x in ends if x > starts[-1]][0]
tot, wtot = defaultdict(float), defaultdict(float)
for n, ms, wgt in seq[s:e + 1]:
    tot[n] += ms
    wtot[n] += ms * wgt
allms, allw = sum(tot.values()), sum(wtot.values())
for n, ms in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{ms:8.3f} ms  {100 * ms / allms:5.1f}%   {wtot[n]:8.3f} SM-weighted ms  {100 * wtot[n] / allw:5.1f}%  {n}")
print(f"{allms:8.3f} ms  step (serialised)   {allw:8.3f} ms SM-weighted")
