"""Summarise one ncu --set full capture: duration, DRAM bytes, pipe/L1/L2
utilisation, top stall reasons and top stalled SASS lines.
    python tools/ncu_summary.py <report.ncu-rep> [ntop]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 16
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u = r[0], r[1]
for v in r[2:]:
    print("==", v[h.index("Kernel Name")][:100])
    for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "sm__warps_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
              "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
              "lts__throughput.avg.pct_of_peak_sustained_elapsed",
              "dram__throughput.avg.pct_of_peak_sustained_elapsed",
              "sm__issue_active.avg.pct_of_peak_sustained_active",
              "launch__registers_per_thread", "launch__grid_size"]:
        if k in h:
            print(f"  {k} = {v[h.index(k)]} {u[h.index(k)]}")
    st = [(h[i], v[i]) for i in range(len(h)) if h[i].startswith("smsp__average_warps_issue_stalled")
          and h[i].endswith("_per_issue_active.ratio")]
    st.sort(key=lambda x: -float(x[1] or 0))
    print("  stalls/issue:", ", ".join(f"{a.split('stalled_')[1].split('_per_issue')[0]}={float(b):.2f}"
                                       for a, b in st[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
if len(rows) > 2:
    hh, data = rows[1], rows[2:]
    si, wi, ai = hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)"), hh.index("Address")
    tot = sum(float(x[wi] or 0) for x in data if len(x) > wi) or 1
    for x in sorted(data, key=lambda x: -float(x[wi] or 0))[:ntop]:
        print(f"  {100 * float(x[wi]) / tot:5.1f}% {x[ai][-5:]} {x[si][:90]}")
