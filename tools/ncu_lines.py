"""Top source lines by warp-stall samples from `ncu -i rep --page source --csv
--print-source cuda,sass` output (profiling tooling).
usage: python tools/ncu_lines.py dump.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, agg, tot = None, [], 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] and r[0].isdigit() and len(r) > 5:
        try:
            s = int(r[4] or 0)
            e = int(r[7] or 0) if len(r) > 7 else 0
        except ValueError:
            continue
        agg.append((s, e, fname, int(r[0]), r[1][:90]))
        tot += s
agg.sort(reverse=True)
print("total samples", tot)
for s, e, f, ln, src in agg[:top]:
    print(f"{100*s/tot:5.1f}% {e:10d} {f}:{ln}  {src}")
