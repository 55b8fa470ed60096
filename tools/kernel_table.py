"""Per-kernel hardware table from an ncu metric capture (test tooling).

Input: the CSV of
  ncu --metrics gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,
        smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,
        dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
      --clock-control none --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu
(three solves: warm-up, re-warm, timed).  Output (JSON, per kernel name, per
solve): launches, serialised ms (ncu runs launches one at a time, cold
cache), executed FP64 thread-instructions (DFMA + DMUL + DADD: one FP64-pipe
slot each), their rate against the FP64 peak of 148 SM x 64 lanes x 1.965
GHz = 1.861e13 slots/s (hw_fp64_frac), DRAM bytes, warp instructions.
usage: python tools/kernel_table.py capture.csv out.json [solves]"""
import csv
import json
import sys
from collections import defaultdict

PEAK_SLOTS = 148 * 64 * 1.965e9

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Name" in r][0]
h = rows[hi]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
solves = int(sys.argv[3]) if len(sys.argv) > 3 else 3
per_launch = defaultdict(dict)
names = {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    lid = int(r[ii])
    names[lid] = r[ki].split("(")[0].replace("void ", "")
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    if r[mi] == "gpu__time_duration.sum":
        v *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}[u]
    elif u in ("Kbyte", "KB"):
        v *= 1e3
    elif u in ("Mbyte", "MB"):
        v *= 1e6
    elif u in ("Gbyte", "GB"):
        v *= 1e9
    per_launch[lid][r[mi]] = v
tab = defaultdict(lambda: defaultdict(float))
for lid, m in per_launch.items():
    t = tab[names[lid]]
    t["launches"] += 1
    t["ms"] += m.get("gpu__time_duration.sum", 0.0)
    t["fp64_slots"] += sum(m.get(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum", 0.0) for op in ("dfma", "dmul", "dadd"))
    t["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    t["warp_inst"] += m.get("smsp__inst_executed.sum", 0.0)
out = {}
for k, t in sorted(tab.items(), key=lambda x: -x[1]["ms"]):
    d = {x: t[x] / solves for x in ("launches", "ms", "fp64_slots", "dram_bytes", "warp_inst")}
    d["hw_fp64_frac"] = d["fp64_slots"] / (d["ms"] / 1e3 * PEAK_SLOTS) if d["ms"] else None
    out[k] = d
json.dump({"source": sys.argv[1], "per_solve": True, "solves": solves, "peak_fp64_slots_per_s": PEAK_SLOTS,
           "kernels": out}, open(sys.argv[2], "w"), indent=1)
for k, d in out.items():
    print(f"{k[:44]:44s} {d['launches']:6.1f} {d['ms']:9.3f} ms  fp64 {d['fp64_slots']:.3e}  hw {d['hw_fp64_frac'] or 0:6.3f}"
          f"  dram {d['dram_bytes'] / 1e9:7.3f} GB")
