"""Per-launch list of the main kernels from an ncu --csv launch list: name:ms(grid)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi, gi = h.index('Kernel Name'), h.index('Metric Value'), h.index('Grid Size')
out, tot = [], {}
for r in rows[hi + 1:]:
    n = r[ki].split('(')[0].replace('void ', '').replace('mrrr::', '').split('<')[0]
    ms = float(r[vi]) / 1e6
    tot[n] = tot.get(n, 0) + ms
    if any(x in n for x in ('refine', 'probe', 'child_warp', 'wvec', 'root_chain', 'k_grid')):
        out.append(f"{n[2:9]}:{ms:.2f}({r[gi].split(',')[0].strip('(')})")
print(' '.join(out))
print('  totals:', {k: round(v, 2) for k, v in sorted(tot.items(), key=lambda x: -x[1])[:6]})
