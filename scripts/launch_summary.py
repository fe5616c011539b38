"""Per-kernel summary of an ncu launch list (gpu__time_duration / dram bytes):
python scripts/launch_summary.py launches.csv [nodes]"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
n = float(sys.argv[2]) if len(sys.argv) > 2 else 113246208
ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
d, names = collections.defaultdict(dict), {}
for r in rows:
    d[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
    names[r[ii]] = r[ki]
agg = collections.defaultdict(list)
for i, m in d.items():
    mm = re.search(r"(\w+_kernel)<(\d+), (\d+)", names[i])
    key = f"{mm.group(1)}<{mm.group(2)},{mm.group(3)}>" if mm else names[i][:50]
    agg[key].append(m)
for k, ms in agg.items():
    busy = [m for m in ms if m.get("gpu__time_duration.sum", 0) > 20000]  # early-exit launches excluded
    if not busy:
        continue
    t = sum(m["gpu__time_duration.sum"] for m in busy) / len(busy) / 1e6
    rd = sum(m.get("dram__bytes_read.sum", 0) for m in busy) / len(busy) / n
    wr = sum(m.get("dram__bytes_write.sum", 0) for m in busy) / len(busy) / n
    print(f"{k:40s} launches={len(busy):3d} ms={t:.3f} read={rd:.1f} B/node write={wr:.1f} B/node "
          f"GB/s={(rd + wr) * n / t / 1e6:.0f}")
