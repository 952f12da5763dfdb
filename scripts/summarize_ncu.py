#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (run here, no GPU needed).

  python scripts/summarize_ncu.py r01

reads gpurun_out/full_<tag>.ncu-rep and gpurun_out/launches_<tag>.csv, writes
profiles/ncu_<tag>.md, profiles/launches_<tag>.csv (kernel, duration) and
profiles/traffic.json (DRAM bytes per launch per kernel, read by bench.py)."""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration_us"),
    ("dram__bytes_read.sum", "dram_read_MB"),
    ("dram__bytes_write.sum", "dram_write_MB"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct_peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_registers", "occ_limit_regs"),
]


def short(name: str) -> str:
    for k in ("forward_tma_kernel", "forward_tile_kernel", "forward_kernel", "merge_follow_kernel", "merge_copy_tma_kernel", "merge_copy_kernel", "merge_scan_kernel",
              "synth_kernel", "set_flags_kernel", "wait_flags_kernel"):
        if k in name:
            return k
    return name.split("(")[0]


def raw_rows(rep: str):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True,
                                  stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def main(tag: str) -> None:
    rep = os.path.join(ROOT, "gpurun_out", f"full_{tag}.ncu-rep")
    hdr, units, rows = raw_rows(rep)
    col = {h: i for i, h in enumerate(hdr)}
    per = defaultdict(list)
    for r in rows:
        k = short(r[col["Kernel Name"]])
        rec = {}
        for m, nice in METRICS:
            if m in col:
                try:
                    rec[nice] = float(r[col[m]].replace(",", ""))
                except ValueError:
                    rec[nice] = r[col[m]]
        # normalise units: ncu reports duration in us (or ns) and bytes in MB (or GB)
        if "gpu__time_duration.sum" in col and units[col["gpu__time_duration.sum"]] == "ns":
            rec["duration_us"] /= 1e3
        for m, nice in (("dram__bytes_read.sum", "dram_read_MB"), ("dram__bytes_write.sum", "dram_write_MB")):
            u = units[col[m]] if m in col else "MB"
            scale = {"byte": 1e-6, "Kbyte": 1e-3, "KB": 1e-3, "Mbyte": 1, "MB": 1, "Gbyte": 1e3, "GB": 1e3}.get(u, 1)
            rec[nice] = rec.get(nice, 0) * scale
        per[k].append(rec)
    lines = [f"# ncu --set full, round tag {tag}",
             "", "Captured with `scripts/profile_round.sh` on one B200 (`--clock-control none`):",
             ("`python bench.py --steps 2 --warmup 3 --profile` (config B, default colocated pass; ncu "
              "serialises the two kernels)" if tag.endswith("_pipe") else
              "`python bench.py --serial --steps 2 --warmup 3 --profile` (config B, 4 requests; K1 "
              "and the merge in stream order, each kernel captured alone)."),
             "Per-launch values; ncu replays each kernel, so durations are cold-cache.", "",
             "| kernel | launches | " + " | ".join(n for _, n in METRICS) + " |",
             "|---|---|" + "---|" * len(METRICS)]
    traffic = {}
    for k, recs in sorted(per.items()):
        avg = {n: sum(r.get(n, 0) for r in recs if isinstance(r.get(n, 0), float)) / len(recs)
               for _, n in METRICS}
        lines.append(f"| {k} | {len(recs)} | " + " | ".join(f"{avg[n]:.3f}" for _, n in METRICS) + " |")
        traffic[k] = round((avg["dram_read_MB"] + avg["dram_write_MB"]) * 1e6)
    lines += ["", "DRAM traffic per launch (read + write) is copied into `profiles/traffic.json`",
              "and reported by bench.py as `roofline.traffic`."]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"ncu_{tag}.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    tr = {"forward_kernel": traffic.get("forward_tma_kernel") or traffic.get("forward_tile_kernel")
          or traffic.get("forward_kernel"),
          "merge": traffic.get("merge_copy_tma_kernel") or traffic.get("merge_copy_kernel"),
          "merge_scan_kernel": traffic.get("merge_scan_kernel"), "source": f"profiles/ncu_{tag}.md",
          "unit": "bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)"}
    if not tag.endswith("_pipe"):
        with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as fh:
            json.dump(tr, fh, indent=1)
    # launch list
    lpath = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    if os.path.exists(lpath):
        txt = open(lpath).read()
        body = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
        rows = list(csv.DictReader(io.StringIO(body)))
        with open(os.path.join(ROOT, "profiles", f"launches_{tag}.csv"), "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["id", "kernel", "metric", "unit", "value"])
            tot = defaultdict(float)
            for r in rows:
                w.writerow([r.get("ID"), short(r.get("Kernel Name", "")), r.get("Metric Name"),
                            r.get("Metric Unit"), r.get("Metric Value")])
                try:
                    tot[short(r.get("Kernel Name", ""))] += float(r.get("Metric Value", "0").replace(",", ""))
                except ValueError:
                    pass
        s = sum(tot.values()) or 1.0
        with open(os.path.join(ROOT, "profiles", f"ncu_{tag}.md"), "a") as fh:
            fh.write("\n## Launch list share (gpu__time_duration.sum, all launches of the run)\n\n")
            fh.write("| kernel | total | share |\n|---|---|---|\n")
            for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
                fh.write(f"| {k} | {v:.1f} | {100 * v / s:.1f}% |\n")
    print(open(os.path.join(ROOT, "profiles", f"ncu_{tag}.md")).read())


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
