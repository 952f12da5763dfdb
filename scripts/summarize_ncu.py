#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (run here, no GPU needed).

  python scripts/summarize_ncu.py r02

reads gpurun_out/full_<tag>_<config>.ncu-rep (+ profile_kernels_<config>.json)
and gpurun_out/launches_<tag>.csv (scripts/profile_round.sh); writes
profiles/ncu_<tag>.md (per-kernel counters, launch-list shares) and
profiles/traffic_<tag>.json: DRAM bytes (read + write) per launch keyed
"<config>:<kernel>" with the launch's algorithmic bytes, which bench.py
reports as `traffic` only for the same kernel on the same launch size."""
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
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]
# kernel -> bench.py's key (kernels.<key>, roofline on the tee)
BENCH_KEY = {"merge_tee_kernel": "tee", "forward_tma_kernel": "forward", "merge_copy_kernel": "merge",
             "merge_follow_kernel": "follow", "merge_scan_kernel": "scan",
             "forward_tile_kernel": "forward_tile"}


def short(name: str) -> str:
    for k in list(BENCH_KEY) + ["synth_kernel", "set_flags_kernel", "wait_flags_kernel", "digest_kernel",
                                "mailbox_kernel", "chan_push_kernel", "chan_pull_kernel"]:
        if k in name:
            return k
    return name.split("(")[0]


def raw_rows(rep: str):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True,
                                  stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def per_kernel(rep: str):
    hdr, units, rows = raw_rows(rep)
    col = {h: i for i, h in enumerate(hdr)}
    per = defaultdict(list)
    for r in rows:
        rec = {}
        for m, nice in METRICS:
            if m in col:
                try:
                    rec[nice] = float(r[col[m]].replace(",", ""))
                except ValueError:
                    rec[nice] = 0.0
        u = units[col["gpu__time_duration.sum"]]
        rec["duration_us"] *= {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1e-3 if u.startswith("n") else 1.0)
        for m, nice in (("dram__bytes_read.sum", "dram_read_MB"), ("dram__bytes_write.sum", "dram_write_MB")):
            scale = {"byte": 1e-6, "Kbyte": 1e-3, "KB": 1e-3, "Mbyte": 1, "MB": 1, "Gbyte": 1e3,
                     "GB": 1e3}.get(units[col[m]], 1)
            rec[nice] *= scale
        per[short(r[col["Kernel Name"]])].append(rec)
    return per


def main(tag: str) -> None:
    lines = [f"# ncu --set full, round tag {tag}", "",
             "Captured with `scripts/profile_round.sh` on one B200 (`--clock-control none`): one launch",
             "of every data-plane kernel on the bench batch (`scripts/profile_kernels.py <config>`:",
             "scan, tee, bulk-copy K1, merge, tile K1, early-start merge with its flags already set).",
             "Per-launch values; ncu replays each kernel, so durations are cold-cache and serialised.", ""]
    traffic = {}
    for config in ("B", "A", "D"):
        rep = os.path.join(ROOT, "gpurun_out", f"full_{tag}_{config}.ncu-rep")
        meta_p = os.path.join(ROOT, "gpurun_out", f"profile_kernels_{config}.json")
        if not os.path.exists(rep):
            continue
        meta = json.load(open(meta_p)) if os.path.exists(meta_p) else {"alg_bytes": {}}
        per = per_kernel(rep)
        lines += [f"## config {config} (payload {meta.get('payload', 0):,} B)", "",
                  "| kernel | launches | " + " | ".join(n for _, n in METRICS) +
                  " | alg MB | DRAM / alg | alg GB/s at ncu time |",
                  "|---|---|" + "---|" * (len(METRICS) + 3)]
        for k, recs in sorted(per.items()):
            avg = {n: sum(r.get(n, 0.0) for r in recs) / len(recs) for _, n in METRICS}
            alg = meta["alg_bytes"].get(k)
            dram = (avg["dram_read_MB"] + avg["dram_write_MB"]) * 1e6
            ratio = f"{dram / alg:.3f}" if alg else "-"
            rate = f"{alg / (avg['duration_us'] * 1e-6) / 1e9:.1f}" if alg and avg["duration_us"] else "-"
            lines.append(f"| {k} | {len(recs)} | " + " | ".join(f"{avg[n]:.3f}" for _, n in METRICS) +
                         f" | {alg / 1e6 if alg else 0:.1f} | {ratio} | {rate} |")
            if alg and k in BENCH_KEY:
                traffic[f"{config}:{BENCH_KEY[k]}"] = {
                    "dram_bytes": round(dram), "alg_bytes": alg, "duration_us": round(avg["duration_us"], 2),
                    "source": f"profiles/ncu_{tag}.md (config {config}, {k})"}
        lines.append("")
    lpath = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    if os.path.exists(lpath):
        txt = open(lpath).read()
        body = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
        rows = list(csv.DictReader(io.StringIO(body)))
        tot = defaultdict(float)
        cnt = defaultdict(int)
        with open(os.path.join(ROOT, "profiles", f"launches_{tag}.csv"), "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["id", "kernel", "metric", "unit", "value"])
            for r in rows:
                k = short(r.get("Kernel Name", ""))
                w.writerow([r.get("ID"), k, r.get("Metric Name"), r.get("Metric Unit"), r.get("Metric Value")])
                try:
                    tot[k] += float(r.get("Metric Value", "0").replace(",", ""))
                    cnt[k] += 1
                except ValueError:
                    pass
        s = sum(tot.values()) or 1.0
        lines += ["## Launch list of `python bench.py --steps 3 --warmup 3 --profile` "
                  "(gpu__time_duration.sum, every launch of the run)", "",
                  "| kernel | launches | total | share |", "|---|---|---|---|"]
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            lines.append(f"| {k} | {cnt[k]} | {v:.1f} | {100 * v / s:.1f}% |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"ncu_{tag}.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    traffic["unit"] = "bytes per launch: dram__bytes_read.sum + dram__bytes_write.sum"
    with open(os.path.join(ROOT, "profiles", f"traffic_{tag}.json"), "w") as fh:
        json.dump(traffic, fh, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
