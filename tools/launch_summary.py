"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys


def summarise(path, title=""):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hdr], rows[hdr + 1:]
    ki, mi, vi, ui = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    scale = {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0][:70]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    tot = sum(v[1] for v in agg.values())
    out = [title] if title else []
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{v[1] / 1e6:9.2f} ms {100 * v[1] / tot:5.1f}%  n={v[0]:5d}  {k}")
    out.append(f"total {tot / 1e6:.2f} ms over {sum(v[0] for v in agg.values())} launches")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1], " ".join(sys.argv[2:])))
