"""Summary of ncu --set full captures (profiling tooling): per launch the
duration, grid, registers, occupancy, issue activity, FP64 pipe, DRAM bytes
and the top stall reasons; then the top source lines by stall samples.
usage: python tools/ncu_summary.py rep.ncu-rep [more.ncu-rep ...]"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum"]

for rep in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    print(f"==== {rep.split('/')[-1]}")
    for v in rows[2:]:
        d = dict(zip(h, v))
        print("----")
        print(f"  {'Kernel Name':70s} {d.get('Kernel Name', '')[:60]}")
        for k in KEYS:
            print(f"  {k:70s} {d.get(k)}")
        st = [(k, float(d[k])) for k in d
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
        st.sort(key=lambda x: -x[1])
        for k, x in st[:6]:
            print(f"  stall {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):30s} {x:.3f}")
