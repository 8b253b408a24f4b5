"""Summarise an ncu source-page CSV (--page source --csv --print-source sass): total executed warp
instructions, the opcode mix, and the main loop (the most executed instruction count) listing.
usage: python scripts/sass_hot.py sass.csv [raw.csv] [--loop]"""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ia = hdr.index('Instructions Executed'); isrc = hdr.index('Source')
tot = 0; op = collections.Counter()
for r in data:
    n = int(r[ia] or 0); tot += n
    m = re.match(r'(@!?U?P\w+\s+)?([A-Z0-9_]+)', r[isrc].strip())
    op[m.group(2) if m else '?'] += n
print('executed warp instructions', tot)
for o, n in op.most_common(16): print(f'  {o:10s} {n:12d} {n / tot * 100:5.1f}%')
cnt = collections.Counter(int(r[ia] or 0) for r in data if 'FMNMX3' in r[isrc])
top = max(c for c, k in cnt.items() if k >= 8)
idx = [i for i, r in enumerate(data) if int(r[ia] or 0) == top]
print('main loop: count', top, 'instructions', len(idx), 'share', len(idx) * top / tot)
if '--loop' in sys.argv:
    for i in range(idx[0], idx[-1] + 1): print(i, data[i][ia], data[i][isrc].strip()[:90])
if len(sys.argv) > 2 and sys.argv[2].endswith('.csv'):
    raw = list(csv.reader(open(sys.argv[2]))); d = dict(zip(raw[0], raw[2]))
    for k in ('gpu__time_duration.sum', 'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed',
              'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
              'sm__warps_active.avg.per_cycle_active'):
        print(' ', k, d.get(k))
