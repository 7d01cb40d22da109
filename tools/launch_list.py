"""Print an ncu --csv gpu__time_duration launch list in launch order (us)."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv")) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
tot = 0.0
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot += v
    print(f"{v:10.1f}  {r[ki][:100]}")
print(f"{tot:10.1f}  total")
