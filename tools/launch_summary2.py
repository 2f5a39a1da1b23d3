"""Per-kernel time / DRAM bytes / fp64-pipe summary of an ncu CSV launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h, data = rows[hdr], rows[hdr + 1:]
ki, ii, mi, vi, ui = (h.index(c) for c in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
per = collections.defaultdict(dict)
names = {}
for r in data:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) if r[vi] else 0.0
    u = r[ui]
    if r[mi] == "gpu__time_duration.sum":
        v *= {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(u, 1)
    if r[mi].startswith("dram__bytes"):
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    per[r[ii]][r[mi]] = v
    names[r[ii]] = r[ki].split("(")[0][:64]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i, m in per.items():
    a = agg[names[i]]
    a[0] += 1
    t = m.get("gpu__time_duration.sum", 0)
    a[1] += t
    a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    a[3] += m.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0) * t
tot = sum(a[1] for a in agg.values())
print(f"{'ms':>8} {'%':>5} {'n':>5} {'GB/s':>7} {'fp64%':>6}  kernel")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{a[1]/1e6:8.2f} {100*a[1]/tot:5.1f} {a[0]:5d} {a[2]/a[1] if a[1] else 0:7.0f} "
          f"{a[3]/a[1] if a[1] else 0:6.1f}  {k}")
print(f"total {tot/1e6:.2f} ms")
