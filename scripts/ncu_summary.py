#!/usr/bin/env python
"""Summarise ncu output brought back in gpurun_out/ into profiles/ (tracked).

  python scripts/ncu_summary.py launches <launches.csv> <out.txt>
  python scripts/ncu_summary.py full <prof.ncu-rep> <out.txt> [--traffic-key KERNEL:CONFIG]

`launches`: per-kernel totals / shares of a `--metrics gpu__time_duration.sum`
launch list (cold-cache, serialised: compare shares, not absolutes).
`full`: key metrics of each kernel in a `--set full` report; with
--traffic-key the per-launch DRAM bytes of the first kernel are written to
profiles/ncu_gs_traffic.json for bench.py's roofline "traffic" field.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "launch__shared_mem_per_block_dynamic", "launch__shared_mem_per_block_static"]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
         "usecond": 1e-3, "msecond": 1.0, "second": 1e3}


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    mi = hdr.index("Metric Name")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    dram = collections.defaultdict(float)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("wd::<unnamed>::", "").replace(
            "wd::(anonymous namespace)::", "")
        if name.startswith("void at::") or name.startswith("at::"):
            name = "[torch input generation / bench glue]"
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            tot[name] += v * SCALE.get(r[ui], 1.0)
            cnt[name] += 1
        elif r[mi].startswith("dram__bytes_"):
            dram[name] += v * SCALE.get(r[ui], 1.0)
    own = sum(v for k, v in tot.items() if not k.startswith("["))
    has_dram = bool(dram)
    lines = [f"# per-kernel device time from {os.path.basename(path)} (ncu gpu__time_duration.sum"
             + (", dram__bytes_read/write.sum" if has_dram else "") +
             ", --clock-control none; cold-cache serialised launches: compare SHARES)",
             f"{'kernel':44s} {'launches':>8s} {'total ms':>10s} {'% of wd':>8s}"
             + (f" {'GB':>9s} {'TB/s':>6s}" if has_dram else "")]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        share = f"{100 * v / own:7.1f}%" if not k.startswith("[") else "     -  "
        ln = f"{k:44s} {cnt[k]:8d} {v:10.3f} {share}"
        if has_dram:
            gb = dram[k] / 1e9
            ln += f" {gb:9.2f} {gb / v if v > 0 else 0:6.2f}"
        lines.append(ln)
    ln = f"{'total wd kernels':44s} {'':8s} {own:10.3f}"
    if has_dram:
        gb = sum(v for k, v in dram.items() if not k.startswith("[")) / 1e9
        ln += f" {'':8s} {gb:9.2f} {gb / own:6.2f}"
    lines.append(ln)
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(path, out, traffic_key=None):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    lines = [f"# key metrics from {os.path.basename(path)} (ncu --set full --clock-control none)"]
    first = None
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        lines.append(f"## {name}")
        d = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"  {k:62s} {r[i]:>16s} {units[i]}")
                try:
                    d[k] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
                except ValueError:
                    pass
        if "dram__bytes_read.sum" in d:
            b = d["dram__bytes_read.sum"] + d.get("dram__bytes_write.sum", 0)
            t = d.get("gpu__time_duration.sum", 0)
            lines.append(f"  {'=> dram bytes per launch':62s} {b:16.0f} byte")
            if t:
                lines.append(f"  {'=> dram GB/s (ncu, cold)':62s} {b / (t * 1e-3) / 1e9:16.1f}")
            if first is None:
                first = b
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_key and first is not None:
        p = os.path.join(ROOT, "profiles", "ncu_gs_traffic.json")
        d = json.load(open(p)) if os.path.exists(p) else {}
        d[traffic_key] = first   # key "<kernel>:<config>" (bench.py reads it)
        json.dump(d, open(p, "w"), indent=1)


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        key = sys.argv[sys.argv.index("--traffic-key") + 1] if "--traffic-key" in sys.argv else None
        full(sys.argv[2], sys.argv[3], key)
