"""The bench's dominant-kernel roofline launch alone (ncu target); with
--write, turn an ncu --set full capture of it into the traffic file bench.py
reads:   python tools/roofline_probe.py [--batch B]
         python tools/roofline_probe.py --write <report.ncu-rep> [--batch B]"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--write", default=None)
a = ap.parse_args()
if a.write:
    from paper_2104_09164_b200.ckks.params import gen_params
    ps = gen_params("fast-hear")
    raw = subprocess.run(["ncu", "-i", a.write, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u, v = r[0], r[1], r[-1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def get(k):
        return float(v[h.index(k)].replace(",", "")) * scale.get(u[h.index(k)], 1)
    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    out = {"kernel": "k_ks3", "tasks": a.batch * (ps.max_level + 2), "n": ps.n,
           "dram_bytes": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
           "duration_under_ncu": v[h.index("gpu__time_duration.sum")] + " " + u[h.index("gpu__time_duration.sum")],
           "source": os.path.basename(a.write)}
    with open(bench.TRAFFIC_FILE, "w") as f:
        json.dump(out, f, indent=1)
    print(out)
else:
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    ps = gen_params("fast-hear")
    be = CkksBackend(ps, seed=0)
    print(bench.dominant_kernel_roofline(be, lvl=ps.max_level, bsz=a.batch, peaks={}))
