"""Summarises an `ncu --page source --csv --print-source=sass` dump: stall
samples by opcode and by barrier-delimited region (diagnostics)."""
import csv
import sys
from collections import defaultdict

r = list(csv.reader(open(sys.argv[1])))
h = r[1]
rows = [x for x in r[2:] if x and x[0] not in ('Address', 'Kernel Name')]
ai, si = h.index('Address'), h.index('Source')
wi, ei = h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed')
ni = h.index('Warp Stall Sampling (Not-issued Samples)')


def f(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


seen, rr = set(), []
for x in rows:
    if x[ai] in seen:
        break
    seen.add(x[ai])
    rr.append(x)
rows = rr
tot = sum(f(x[wi]) for x in rows)
print('samples', tot, 'instructions', len(rows))
ops = defaultdict(float)
for x in rows:
    t = x[si].split()
    if t:
        ops[(t[1] if t[0].startswith('@') else t[0]).split('.')[0]] += f(x[wi])
print(' '.join(f'{k}={v / tot * 100:.1f}%' for k, v in sorted(ops.items(), key=lambda t: -t[1])[:12]))
stall_cols = [i for i, k in enumerate(h) if k.startswith('stall_') and 'Not Issued' not in k]
cuts = sorted(set([0, len(rows)] + [i for i, x in enumerate(rows) if 'BAR.SYNC' in x[si] or 'BAR.SYNC' in x[si]]
                  + [int(a) for a in sys.argv[2:]]))
for a, b in zip(cuts[:-1], cuts[1:]):
    s = sum(f(x[wi]) for x in rows[a:b])
    if s / tot < 0.01:
        continue
    st = sorted(((sum(f(x[i]) for x in rows[a:b]), h[i][6:]) for i in stall_cols), reverse=True)[:5]
    fp = sum(f(x[ei]) for x in rows[a:b] if any(o in x[si] for o in ('FFMA2', 'FMUL2', 'FADD2')))
    ex = sum(f(x[ei]) for x in rows[a:b])
    print(f'[{a},{b}) {s / tot * 100:5.1f}%  instr {ex / 1e6:.1f}M fp32x2 {fp / 1e6:.1f}M  ' +
          ' '.join(f'{k}={v / s * 100:.0f}%' for v, k in st) + f'  | {rows[a][si][:40]}')
