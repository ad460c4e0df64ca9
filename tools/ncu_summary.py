"""Summarise one `ncu --set full` capture of the pair kernel into
profiles/traffic.json (read by bench.py for roofline.traffic and the pipe
utilisation):  python tools/ncu_summary.py REP.ncu-rep WORKLOAD N DETAILS_CSV"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
           "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "smsp__inst_executed.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

rep, wl, n, details = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]
m = {k: {"value": v[h.index(k)], "unit": units[h.index(k)]} for k in METRICS if k in h}
tb = sum(float(m[k]["value"]) * SCALE[m[k]["unit"]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
doc = json.load(open(path)) if os.path.exists(path) else {}
doc[wl] = {"n": n, "capture": details, "kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else "",
           "bytes_per_launch": tb, "metrics": m}
json.dump(doc, open(path, "w"), indent=1)
print(wl, tb, {k: m[k]["value"] for k in m})
