"""Summarise ncu output into profiles/ (launch list shares + full-set metrics).

  python tools/ncu_summary.py <launches.csv> <prof.ncu-rep> <tag>
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
    "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
]


def launches(path):
    text = open(path).read()
    lines = text.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"') or l.startswith("ID"))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    per = defaultdict(list)
    for r in rows:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            name = r["Kernel Name"].split("(")[0]
            v = float(r["Metric Value"].replace(",", ""))
            unit = r.get("Metric Unit", "ns")
            scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3,
                     "msecond": 1e3}.get(unit, 1.0)
            per[name].append(v * scale)
    tot = sum(sum(v) for v in per.values())
    out = ["kernel | launches | avg us | share of GPU time", "---|---|---|---"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{k} | {len(v)} | {sum(v)/len(v):.1f} | {100*sum(v)/tot:.1f}%")
    return "\n".join(out), per


def full(rep):
    """rep: a .ncu-rep, or the CSV of `ncu -i rep --page raw --csv`; several
    may be joined with commas (each parsed with its own header)."""
    res = []
    for part in rep.split(","):
        if part.endswith(".csv"):
            raw = open(part).read()
        else:
            raw = subprocess.run(["ncu", "-i", part, "--page", "raw", "--csv"],
                                 capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            d = {"kernel": r[hdr.index("Kernel Name")]}
            for m in METRICS:
                if m in hdr:
                    d[m] = f"{r[hdr.index(m)]} {units[hdr.index(m)]}".strip()
            res.append(d)
    return res


def main():
    """ncu_summary.py <launches.csv> <raw.csv[,raw.csv...]> <tag> [launch-list command]"""
    lpath, rep, tag = sys.argv[1:4]
    cmd = sys.argv[4] if len(sys.argv) > 4 else (
        "python bench.py --steps 2 --warmup 3 --e2e-steps 2 --no-cpu-baseline")
    table, per = launches(lpath)
    kern = full(rep)
    with open(os.path.join(PROF, f"{tag}_launches.md"), "w") as fh:
        fh.write(f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)\n\n")
        fh.write(f"Command: `{cmd}` (C3, FP64). Times are cold-cache and serialised: compare "
                 "shares, not absolutes.\n\n")
        fh.write(table + "\n")
    with open(os.path.join(PROF, f"{tag}_ncu_full.md"), "w") as fh:
        fh.write(f"# {tag}: ncu --set full\n\n"
                 "One launch per kernel (-c 1 after warm-up launches), --clock-control none, cold "
                 "cache; targets in tools/probe.py (`ncu pair`: C3 pairs; `ncu gradient`: C4 "
                 "one-shot; `ncu aa`: C3 in-place pairs).\n\n")
        for d in kern:
            fh.write(f"## {d['kernel']}\n\n")
            for m in METRICS:
                if m in d:
                    fh.write(f"- {m}: {d[m]}\n")
            fh.write("\n")
    # DRAM bytes per launch (bench.py's roofline.traffic reads the k_pair entry)
    tj = {}
    for d in kern:
        def val(m):
            v, u = d[m].split(" ")[0].replace(",", ""), d[m].split(" ")[1] if " " in d[m] else ""
            return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        b = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        name = d["kernel"].split("(")[0].split("<")[0].split()[-1].split("::")[-1]
        key = "pair_bytes_per_launch" if name == "k_pair" else f"{name}_bytes_per_launch"
        tj[key] = b
    tj["source"] = f"profiles/{tag}_ncu_full.md (ncu --set full)"
    with open(os.path.join(PROF, "traffic.json"), "w") as fh:
        json.dump(tj, fh, indent=1)
    print(table)
    print(json.dumps(tj, indent=1))


if __name__ == "__main__":
    main()
