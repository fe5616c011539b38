"""Summarise gpurun_out ncu artefacts into text for profiles/.

    python scripts/summarize_ncu.py gpurun_out/<tag> profiles/<round>_<tag>.txt

Reads launches.csv (ncu --metrics gpu__time_duration.sum launch list),
prof_pr.ncu-rep / prof_ffg.ncu-rep (full or sectioned captures) and bench.json.
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

KEYS = ("Duration", "DRAM Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput",
        "Compute (SM) Throughput", "Memory Throughput", "L2 Hit Rate", "Achieved Occupancy",
        "Registers Per Thread", "Warp Cycles Per Issued Instruction", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct")


def ncu(*args) -> str:
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def launches(path: str) -> list[str]:
    lines = [l for l in open(path) if l.startswith('"')]
    agg = defaultdict(list)
    for r in csv.DictReader(lines):
        agg[r["Kernel Name"].split("(")[0]].append(float(r["Metric Value"]) / 1e6)
    total = sum(sum(v) for v in agg.values())
    out = ["kernel | launches | mean ms | share of listed time"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{k[-60:]} | {len(v)} | {sum(v) / len(v):.3f} | {100 * sum(v) / total:.1f}%")
    return out


def details(rep: str) -> list[str]:
    txt = ncu("-i", rep, "--page", "details", "--csv")
    out = []
    for row in csv.reader(io.StringIO(txt)):
        if len(row) < 4:
            continue
        if row[0] == "ID":
            continue
        name = row[4] if len(row) > 4 else ""
        metric, unit, value = row[-3], row[-2], row[-1]
        if metric in KEYS:
            out.append(f"{metric}: {value} {unit}".rstrip())
        if metric == "Duration" and name:
            out.insert(0, f"kernel: {name[:120]}")
    return out


def stalls(rep: str, top: int = 12) -> list[str]:
    txt = ncu("-i", rep, "--page", "source", "--csv")
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return []
    h, data = rows[1], rows[2:]
    try:
        i_s = h.index("Warp Stall Sampling (All Samples)")
    except ValueError:
        return []
    cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    agg = {h[i]: sum(int(r[i]) for r in data if r[i].isdigit()) for i in cols}
    tot = sum(agg.values()) or 1
    out = ["stall reasons (share of samples): " + ", ".join(
        f"{k[6:]} {100 * v / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:6])]
    out.append("top SASS lines by samples:")
    for r in sorted(data, key=lambda r: -int(r[i_s]) if r[i_s].isdigit() else 0)[:top]:
        st = sorted(((int(r[i]), h[i][6:]) for i in cols if r[i].isdigit()), reverse=True)[:2]
        out.append(f"  {r[i_s]:>8}  {r[1].strip()[:60]:<60} {st}")
    return out


def main(src: str, dst: str) -> None:
    out = [f"# ncu / bench summary of {src}", ""]
    b = os.path.join(src, "bench.json")
    if os.path.exists(b):
        d = json.load(open(b))
        out += ["## bench.py line", json.dumps(d, indent=1), ""]
    if os.path.exists(os.path.join(src, "launches.csv")):
        out += ["## launch list (ncu gpu__time_duration.sum; cold-cache, serialised)"]
        out += launches(os.path.join(src, "launches.csv")) + [""]
    for name in ("prof_pr", "prof_ffg"):
        rep = os.path.join(src, name + ".ncu-rep")
        if os.path.exists(rep):
            out += [f"## {name}"] + details(rep) + stalls(rep) + [""]
    os.makedirs(os.path.dirname(dst) or ".", exist_ok=True)
    with open(dst, "w") as f:
        f.write("\n".join(out) + "\n")
    print(dst)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
