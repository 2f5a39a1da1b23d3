"""Dynamic SASS opcode mix (instructions executed) of an ncu capture made
with --import-source on.   python tools/ncu_opmix.py <report.ncu-rep> [elements]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
elems = float(sys.argv[2]) if len(sys.argv) > 2 else 0
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h, data = rows[1], rows[2:]
si, ie = h.index("Source"), h.index("Instructions Executed")
wi = h.index("Warp Stall Sampling (All Samples)")
cnt, st = collections.Counter(), collections.Counter()
for r in data:
    op = r[si].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    o = o.split(".")[0]
    cnt[o] += float(r[ie] or 0)
    st[o] += float(r[wi] or 0)
tot, stot = sum(cnt.values()), sum(st.values()) or 1
for o, c in cnt.most_common(24):
    per = f"{32 * c / elems:7.2f}/elem" if elems else ""
    print(f"{o:10s} {c / 1e6:9.2f}M {100 * c / tot:5.1f}%  {per}  stall {100 * st[o] / stot:5.1f}%")
print(f"total {tot / 1e6:.2f}M warp instructions" + (f", {32 * tot / elems:.1f} per element" if elems else ""))
