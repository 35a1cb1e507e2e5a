"""Summarise a tools/profile_round.sh capture into profiles/<round>/:
launch-list shares, ncu --set full per-kernel table (time, DRAM bytes, DRAM %
of peak, warps / issue active, registers, top stalls) and the aggregation
stage's DRAM bytes per step (agg_traffic.json, read by bench.py).

    python tools/profile_summary.py TAG OUTDIR BATCH TEXTURE_SCALE
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

tag, outdir, batch, tex = sys.argv[1], sys.argv[2], int(sys.argv[3]), float(sys.argv[4])
src = "gpurun_out"
os.makedirs(outdir, exist_ok=True)
lines = []

# ---- launch list
rows = [r for r in csv.reader(open(f"{src}/prof_{tag}_launches.csv")) if r and not r[0].startswith("==")]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("es::", "")
    v = float(r[vi].replace(",", ""))
    unit = r[hdr.index("Metric Unit")]
    ms = v / 1e6 if unit == "ns" else (v / 1e3 if unit == "us" else (v if unit == "ms" else v / 1e6))
    tot[name] += ms
    cnt[name] += 1
allms = sum(v for k, v in tot.items() if "render" not in k)
lines.append(f"## Launch list `{tag}` (`ncu --metrics gpu__time_duration.sum --clock-control none`, "
             f"bench --steps 2 --warmup 3 --batch {batch}: all launches incl. warm-up and frame 0)\n")
lines.append("| kernel | launches | ms (sum) | share (excl. render) |\n|---|---|---|---|")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    share = "" if "render" in k else f"{100 * v / allms:.1f}%"
    lines.append(f"| {k} | {cnt[k]} | {v:.2f} | {share} |")
lines.append("")

# ---- ncu full (one timed step)
raw = subprocess.run(["ncu", "-i", f"{src}/prof_{tag}_full.ncu-rep", "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
lines.append(f"## ncu --set full, one timed step (B={batch}), `{tag}`\n")
lines.append("| kernel | ms | DRAM GB | DRAM % peak | warps active % | issue active % | regs | top stalls (cycles per issue) |")
lines.append("|---|---|---|---|---|---|---|---|")
agg_bytes, agg_ms, agg_alu = 0.0, 0.0, 0.0
per_kernel = {}   # ncu DRAM bytes, ms and ALU-pipe share of the other hot kernels
table = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("es::", "")
    ms = float(d["gpu__time_duration.sum"])
    dram = float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"])
    unit = rows[1][hdr.index("dram__bytes_read.sum")]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    dram *= scale
    if "grp4" in name:
        agg_bytes += dram
        agg_ms += ms
        agg_alu += ms * float(d["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"])
    st = {k: float(v) for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled")
          and k.endswith("per_issue_active.ratio") and v}
    top = ", ".join("%s %.1f" % (k.replace("smsp__average_warps_issue_stalled_", "").replace(
        "_per_issue_active.ratio", ""), v) for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
    if ms < 0.05:
        continue   # early-exit regime variants
    for key, pat in (("cost", "k_cost_runs"), ("wta_variance", "k_wta_runs")):
        if pat in name:
            per_kernel[key] = {"dram_bytes_per_step": dram, "ms_serialised": ms,
                               "alu_pipe_active_pct": float(d["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"])}
    lines.append(f"| {name} | {ms:.2f} | {dram / 1e9:.2f} | {float(d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']):.1f} | "
                 f"{float(d['sm__warps_active.avg.pct_of_peak_sustained_active']):.1f} | "
                 f"{float(d['smsp__issue_active.avg.pct_of_peak_sustained_active']):.1f} | "
                 f"{d['launch__registers_per_thread']} | {top} |")
lines.append("")
lines.append(f"Aggregation stage (k_sgm_grp4 launches of the step): {agg_ms:.2f} ms serialised, "
             f"{agg_bytes / 1e9:.2f} GB DRAM.\n")
with open(os.path.join(outdir, f"SUMMARY_{tag}.md"), "w") as fh:
    fh.write("\n".join(lines) + "\n")
json.dump({"batch": batch, "texture_scale": tex, "config": 5, "dram_bytes_per_step": agg_bytes,
           "kernel_ms_per_step_serialised": agg_ms,
           "alu_pipe_active_pct": agg_alu / agg_ms if agg_ms else None,
           "stages": per_kernel,
           "alu_source": "time-weighted sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active "
                         "over the same k_sgm_grp4 launches",
           "source": f"profiles/r01/SUMMARY_{tag}.md: sum of dram__bytes_read.sum + dram__bytes_write.sum "
                     f"over the k_sgm_grp4 launches of one timed step (ncu --set full)"},
          open(os.path.join(outdir, "agg_traffic.json"), "w"), indent=1)
print("\n".join(lines))
