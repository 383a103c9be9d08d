"""Brief per-kernel summary of an ncu report: time, DRAM bytes, issue/pipe utilisation, top stalls.
    python tools/ncu_brief.py gpurun_out/x.ncu-rep"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
want = {"gpu__time_duration.sum": "us", "dram__bytes_read.sum": "rd", "dram__bytes_write.sum": "wr",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "warps%",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu%",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma%",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu%",
        "launch__registers_per_thread": "regs", "sm__inst_executed.sum": "inst",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram%"}
for v in rows[2:]:
    name = v[h.index("Kernel Name")][:60]
    out = {}
    for i, k in enumerate(h):
        if k in want:
            out[want[k]] = v[i]
    st = []
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v[i]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    st.sort(reverse=True)
    print(name, out, "stalls:", ", ".join(f"{n} {x:.2f}" for x, n in st[:6]))
