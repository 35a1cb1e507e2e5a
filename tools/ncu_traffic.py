"""Measure the DRAM traffic and pipe usage of one bench step per stage with
ncu and record it, stamped with the library's SHA-256, in
profiles/ncu_traffic.json (bench.py reports these numbers only for the
same library build).  Run on the GPU box from the repo root:

    python tools/ncu_traffic.py [--batch 64] [--config 5] [--tag r02]

ncu replays every kernel of `bench.py --steps 1 --warmup 3` with a small
metric set; the step used is the last complete one (the timed step).  The
per-launch numbers are cold-cache and serialised -- the bench line uses
them for bytes moved, never for time.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
# kernel name -> bench stage (es_ctx_stage_times order)
STAGES = [("k_warp_zmax", "predict"), ("k_warp_zidx", "predict"), ("k_resolve_fill_h", "predict"),
          ("k_fill_v_intervals", "intervals"), ("k_cost_runs", "cost"), ("k_sgm_", "aggregate"),
          ("k_wta_runs", "wta_variance"), ("k_checks_fuse", "checks_fuse")]
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3,
         "ns": 1e-6, "us": 1e-3, "ms": 1.0,
         "msecond": 1.0, "%": 1, "inst": 1, "": 1}


def lib_sha256():
    """Build id of the kernels (sources + flags; see build.build_id)."""
    sys.path.insert(0, ROOT)
    from paper_1708_06301_b200 import build as _b
    return _b.build_id()


def merge(entry):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        entries = json.load(open(path))
    except (OSError, ValueError):
        entries = []
    entries = [x for x in entries if not (x.get("lib_sha256") == entry["lib_sha256"]
                                          and x.get("config") == entry["config"]
                                          and x.get("batch") == entry["batch"])]
    entries.append(entry)
    json.dump(entries, open(path, "w"), indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--tag", default="r02")
    ap.add_argument("--merge", default=None,
                    help="(build container) merge a gpurun_out/ncu_traffic_TAG.json entry into "
                         "profiles/ncu_traffic.json")
    args = ap.parse_args()
    if args.merge:
        merge(json.load(open(args.merge)))
        return
    out_csv = os.path.join(ROOT, "gpurun_out", f"ncu_traffic_{args.tag}.csv")
    os.makedirs(os.path.dirname(out_csv), exist_ok=True)
    cmd = ["ncu", "--metrics", ",".join(METRICS), "--clock-control", "none", "--csv",
           "-k", "regex:^k_", "--log-file", out_csv,
           sys.executable, "bench.py", "--steps", "1", "--warmup", "3", "--no-cpu", "--no-e2e",
           "--config", str(args.config), "--batch", str(args.batch)]
    subprocess.run(cmd, cwd=ROOT, check=True, stdout=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(open(out_csv).read())))
    hdr = None
    launches = defaultdict(dict)   # ID -> {metric: value, name}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            lid = int(d["ID"])
            launches[lid]["name"] = d["Kernel Name"].split("(")[0].replace("void ", "")
            try:
                v = float(d["Metric Value"].replace(",", ""))
            except ValueError:
                continue
            launches[lid][d["Metric Name"]] = v * UNITS.get(d["Metric Unit"], 1)
    seq = [launches[i] for i in sorted(launches)]
    starts = [i for i, L in enumerate(seq) if "k_warp_zmax" in L["name"]]
    ends = [i for i, L in enumerate(seq) if "k_checks_fuse" in L["name"]]
    # B >= 64 runs as several contexts (BatchedPipeline groups), each
    # launching a whole step: the last step is the last `groups` context steps
    sys.path.insert(0, ROOT)
    from paper_1708_06301_b200.pipeline import default_groups
    groups = default_groups(args.batch)
    s = starts[-groups]
    e = ends[-1]
    stages = defaultdict(lambda: {"dram_bytes_per_step": 0.0, "ms_serialised": 0.0,
                                  "alu_weighted": 0.0, "instructions": 0.0, "launches": 0})
    kernels = defaultdict(lambda: {"dram_bytes": 0.0, "ms": 0.0, "launches": 0})
    for L in seq[s:e + 1]:
        stage = next((st for pat, st in STAGES if pat in L["name"]), None)
        if stage is None:
            continue
        dram = L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0)
        ms = L.get("gpu__time_duration.sum", 0)
        st = stages[stage]
        st["dram_bytes_per_step"] += dram
        st["ms_serialised"] += ms
        st["alu_weighted"] += ms * L.get("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 0)
        st["instructions"] += L.get("smsp__inst_executed.sum", 0)
        st["launches"] += 1
        k = kernels[L["name"].replace("es::", "")]
        k["dram_bytes"] += dram
        k["ms"] += ms
        k["launches"] += 1
    out_stages = {}
    for name, st in stages.items():
        out_stages[name] = {"dram_bytes_per_step": st["dram_bytes_per_step"],
                            "ms_serialised": st["ms_serialised"],
                            "alu_pipe_active_pct": st["alu_weighted"] / st["ms_serialised"]
                            if st["ms_serialised"] else None,
                            "warp_instructions": st["instructions"], "launches": st["launches"]}
    entry = {"lib_sha256": lib_sha256(), "config": args.config, "batch": args.batch,
             "texture_scale": 0.05, "tag": args.tag, "stages": out_stages,
             "kernels": dict(kernels),
             "capture": " ".join(os.path.basename(c) for c in cmd) + " (last complete step)"}
    merge(entry)
    # the copy that comes back with gpurun (merge it here with --merge)
    json.dump(entry, open(os.path.join(ROOT, "gpurun_out", f"ncu_traffic_{args.tag}.json"), "w"),
              indent=1)
    for name, st in sorted(out_stages.items(), key=lambda kv: -kv[1]["ms_serialised"]):
        print(f"{name:14s} {st['ms_serialised']:8.3f} ms  {st['dram_bytes_per_step'] / 1e9:7.2f} GB  "
              f"ALU {st['alu_pipe_active_pct'] or 0:5.1f}%")


if __name__ == "__main__":
    main()
