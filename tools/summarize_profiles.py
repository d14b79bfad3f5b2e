"""Summarise ncu output into profiles/ (committed evidence).

    python tools/summarize_profiles.py <round-tag> <launches.csv> <full.ncu-rep> [more.ncu-rep ...]
        [--config K --cells M --cmd "..."]

Writes profiles/<tag>_launches.md (per-kernel launch count, time share from the
cold-cache serialised launch list), profiles/<tag>_ncu_full.md (DRAM bytes,
throughput, occupancy and stall reasons per kernel from one --set full
capture) and profiles/ncu_summary_<tag>.json (read by bench.py for the
roofline `traffic` field).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name):
    n = name.split("(")[0].replace("void ", "").replace("tmg::", "")
    return n.split("<")[0]


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    agg = defaultdict(lambda: [0, 0.0])  # launches, ns
    for r in rows[start + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        k = short(r[ki])
        agg[k][0] += 1
        agg[k][1] += float(r[vi].replace(",", "")) * TSCALE_NS.get(r[ui] if ui is not None else "nsecond", 1)
    return agg


TSCALE_NS = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
             "second": 1e9, "s": 1e9}


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        k = short(r[hdr.index("Kernel Name")])
        g = lambda m: float(r[hdr.index(m)]) if m in hdr and r[hdr.index(m)] not in ("", "n/a") else None
        u = lambda m: units[hdr.index(m)] if m in hdr else ""
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = g("dram__bytes_read.sum") * scale.get(u("dram__bytes_read.sum"), 1)
        wr = g("dram__bytes_write.sum") * scale.get(u("dram__bytes_write.sum"), 1)
        tus = g("gpu__time_duration.sum") * TSCALE_NS.get(u("gpu__time_duration.sum"), 1e3) * 1e-3
        st = sorted(((hdr[i].replace("smsp__average_warps_issue_stalled_", "").replace(
            "_per_issue_active.ratio", ""), float(r[i])) for i in range(len(hdr))
            if hdr[i].startswith("smsp__average_warps_issue_stalled_")
            and hdr[i].endswith("per_issue_active.ratio") and r[i] not in ("", "n/a")),
            key=lambda x: -x[1])[:4]
        res.setdefault(k, {
            "duration_us": tus, "dram_bytes_per_launch": rd + wr,
            "dram_read_bytes": rd, "dram_write_bytes": wr,
            "dram_pct_peak": g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "achieved_gbs": (rd + wr) / (tus * 1e-6) / 1e9 if tus else None,
            "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "registers": g("launch__registers_per_thread"),
            "top_stalls": [(a, round(b, 2)) for a, b in st],
        })
    return res


def main():
    argv = list(sys.argv[1:])
    opt = {}
    for key in ("--config", "--cells", "--cmd"):
        if key in argv:
            i = argv.index(key)
            opt[key] = argv[i + 1]
            del argv[i:i + 2]
    tag, lpath, fpaths = argv[0], argv[1], argv[2:]
    cfg = int(opt.get("--config", 1))
    cells = int(opt.get("--cells", 128 ** 3))
    cmd = opt.get("--cmd", "python bench.py --config 1 --steps 1 --warmup 3 --no-cpu-baseline --no-extra")
    size = f"{round(cells ** (1 / 3))}^3"
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    agg = launches(lpath)
    tot = sum(v[1] for v in agg.values())
    with open(os.path.join(prof, f"{tag}_launches.md"), "w") as f:
        f.write(f"# {tag}: ncu launch list (`--metrics gpu__time_duration.sum --clock-control none`)\n\n")
        f.write(f"Command: `{cmd}` (BASELINE configs[{cfg}], {size}: set-up + solves). "
                "Cold-cache, serialised per-launch times: compare shares, not absolutes.\n\n")
        f.write("| kernel | launches | total us | share |\n|---|---:|---:|---:|\n")
        for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"| {k} | {n} | {t / 1e3:.1f} | {100 * t / tot:.1f}% |\n")
    fr = {}
    for fp in fpaths:
        for k, v in full(fp).items():
            fr.setdefault(k, v)
    with open(os.path.join(prof, f"{tag}_ncu_full.md"), "w") as f:
        f.write(f"# {tag}: ncu --set full (one launch per kernel, configs[{cfg}] {size})\n\n")
        f.write("| kernel | us | DRAM MB/launch | achieved GB/s | DRAM % peak | warps active % | regs | top stalls |\n")
        f.write("|---|---:|---:|---:|---:|---:|---:|---|\n")
        for k, v in fr.items():
            f.write(f"| {k} | {v['duration_us']:.1f} | {v['dram_bytes_per_launch'] / 1e6:.1f} | "
                    f"{(v['achieved_gbs'] or 0):.0f} | {v['dram_pct_peak'] or 0:.1f} | "
                    f"{v['warps_active_pct'] or 0:.1f} | {v['registers'] or 0:.0f} | {v['top_stalls']} |\n")
    with open(os.path.join(prof, f"ncu_summary_{tag}.json"), "w") as f:
        json.dump({"tag": tag, "config": cfg, "cells": cells, "command": cmd, "kernels": fr,
                   "launch_share": {k: {"launches": n, "total_us": t / 1e3, "share": t / tot}
                                    for k, (n, t) in agg.items()}}, f, indent=1)
    print(open(os.path.join(prof, f"{tag}_launches.md")).read())
    print(open(os.path.join(prof, f"{tag}_ncu_full.md")).read())


if __name__ == "__main__":
    main()
