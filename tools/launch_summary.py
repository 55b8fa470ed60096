"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; data = rows[hi + 1:]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
idi = h.index('ID') if 'ID' in h else None
scale = {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0, 'msecond': 1.0}
per = [(r[ki].split('(')[0].replace('void ', ''), float(r[vi].replace(',', '')) * scale[r[ui]]) for r in data if len(r) > vi]
nsolve = int(sys.argv[2]) if len(sys.argv) > 2 else 1
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
per = per[skip:]
tot = defaultdict(float); cnt = defaultdict(int)
for k, v in per:
    tot[k] += v; cnt[k] += 1
T = sum(tot.values())
print(f"{'kernel':60s} {'launches':>8s} {'ms/solve':>10s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k[:60]:60s} {cnt[k]/nsolve:8.1f} {v/nsolve:10.3f} {100*v/T:6.2f}%")
print(f"total launches {len(per)}  kernel ms/solve {T/nsolve:.2f}")
