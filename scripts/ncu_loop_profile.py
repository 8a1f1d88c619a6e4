"""Summarise an ncu --set full capture (raw.csv + src.csv exported with
--page raw/source --csv): headline metrics, stall mix, and the sample
distribution along the SASS of the kernel in chunks of 20 instructions."""
import csv, sys
from collections import Counter
raw, src = sys.argv[1], sys.argv[2]
lo = int(sys.argv[3]) if len(sys.argv) > 3 else 0
rows = list(csv.reader(open(raw)))
d = dict(zip(rows[0], rows[2]))
keys = ['gpu__time_duration.sum', 'smsp__inst_executed.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__cycles_elapsed.max', 'launch__registers_per_thread', 'launch__grid_size']
print({k: d[k] for k in keys})
print('stalls', {k.split('issue_stalled_')[1].split('_per')[0]: round(float(x), 2) for k, x in d.items()
                 if 'issue_stalled' in k and 'per_issue_active' in k and float(x) > 0.15})
rows = list(csv.reader(open(src)))
h = rows[1]; data = rows[2:]; ix = {x: i for i, x in enumerate(h)}
S = lambda r: int(r[ix['# Samples']] or 0)
I = lambda r: int(r[ix['Instructions Executed']] or 0)
tot = sum(S(r) for r in data)
grid = int(d['launch__grid_size'])
print('lines', len(data), 'samples', tot, 'warp-instr per patch', sum(I(r) for r in data) / grid)
for c0 in range(lo, len(data), 20):
    ch = data[c0:c0 + 20]
    s_ = sum(S(r) for r in ch)
    if s_ < 0.004 * tot:
        continue
    ops = Counter((r[ix['Source']].split()[1] if r[ix['Source']].startswith('@') else r[ix['Source']].split()[0]) for r in ch)
    st = Counter()
    for r in ch:
        for k in h:
            if k.startswith('stall_') and 'Not' not in k:
                st[k[6:]] += int(r[ix[k]] or 0)
    print(f'{c0:5d} smp {s_/tot:6.3f} inst/patch {sum(I(r) for r in ch)/grid:8.0f} {ops.most_common(3)} {st.most_common(3)}')
