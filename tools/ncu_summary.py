"""Summarise one `ncu --set full` capture of the pair kernel into
profiles/traffic.json (read by bench.py for roofline.traffic and the binding
pipe):  python tools/ncu_summary.py REP.ncu-rep WORKLOAD N DETAILS_CSV [PAIRS_PER_LAUNCH]

Keeps the DRAM bytes, duration, SM clock, issue / pipe utilisations and
instruction counts of the captured launch, plus the hash of the device
source it was built from (bench.py attributes a capture only to a run of the
same kernel source)."""
import csv
import hashlib
import io
import json
import os
import subprocess
import sys

KEEP_PREFIX = ("gpu__time_duration", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__issue_active",
               "sm__pipe_", "sm__inst_executed_pipe_", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
               "l1tex__data_pipe_lsu_wavefronts_mem_shared", "sm__warps_active", "launch__registers_per_thread",
               "launch__occupancy_limit", "sm__throughput", "smsp__average_warps_issue_stalled")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

rep, wl, n, details = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
pairs = int(sys.argv[5]) if len(sys.argv) > 5 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, kernels = rows[0], rows[1], [r for r in rows[2:] if len(r) == len(rows[0])]


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


# several captured launches (e.g. the two size classes / plans of one step):
# durations and counts add up, utilisations are duration-weighted means
it = h.index("gpu__time_duration.sum")
ia = h.index("smsp__inst_executed.sum")
# a launch ncu could time but not replay reports nan metrics: only its
# duration is kept (other_time), the metrics come from the replayed launches
other = [r for r in kernels if num(r[ia]) is None or num(r[ia]) != num(r[ia])]
other_time = sum(num(r[it]) or 0.0 for r in other)
kernels = [r for r in kernels if r not in other] or kernels
dur = [num(r[it]) or 0.0 for r in kernels]
m = {}
for i, k in enumerate(h):
    if not k.startswith(KEEP_PREFIX):
        continue
    vals = [num(r[i]) for r in kernels]
    if len(kernels) == 1 or any(x is None for x in vals):
        m[k] = {"value": kernels[0][i], "unit": units[i]}
    elif k.endswith(".sum") and "pct" not in k and "per_second" not in k:
        m[k] = {"value": repr(sum(vals)), "unit": units[i]}
    else:
        m[k] = {"value": repr(sum(x * d for x, d in zip(vals, dur)) / max(sum(dur), 1e-30)), "unit": units[i]}
tb = sum(float(m[k]["value"].replace(",", "")) * SCALE[m[k]["unit"]]
         for k in ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in m)
v = kernels[0]
sha = hashlib.sha1(open(os.path.join(ROOT, "paper_2410_04349_b200", "csrc", "rb_device.cuh"), "rb").read()).hexdigest()[:12]
path = os.path.join(ROOT, "profiles", "traffic.json")
doc = json.load(open(path)) if os.path.exists(path) else {}
doc[wl] = {"n": n, "capture": details, "launches": len(kernels), "other_launches": len(other),
           "other_time": other_time, "time_unit": units[it],
           "kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else "",
           "kernel_sha": sha, "pairs": pairs, "bytes_per_launch": tb, "metrics": m}
json.dump(doc, open(path, "w"), indent=1)
print(wl, tb, len(m), "metrics kept")
