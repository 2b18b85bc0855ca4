#!/usr/bin/env python
"""Bucket an ncu --page source --csv dump into contiguous SASS regions split
at lines whose execution count changes by > 20 %, and print stall samples by
reason per region (where the kernel spends its warp-cycles)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
iS = h.index('Warp Stall Sampling (All Samples)')
iE = h.index('Instructions Executed')
reasons = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
ri = [h.index(c) for c in reasons]
tot = sum(int(r[iS]) for r in data) or 1
regions = []
cur = None
for r in data:
    e = int(r[iE])
    if cur is None or (e and abs(e - cur['e']) > 0.2 * max(e, cur['e'])):
        cur = {'e': e, 'start': r[0][-5:], 'first': r[1][:40], 'n': 0, 'S': 0,
               'R': [0] * len(ri), 'I': 0}
        regions.append(cur)
    cur['n'] += 1
    cur['S'] += int(r[iS])
    cur['I'] += e
    for k, i in enumerate(ri):
        cur['R'][k] += int(r[i] or 0)
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
for g in regions:
    if g['S'] < thr * tot:
        continue
    top = sorted(zip(g['R'], reasons), reverse=True)[:4]
    print(f"{g['start']} n={g['n']:4d} exec={g['e']:>11d} samples {100*g['S']/tot:5.1f}%  "
          + ", ".join(f"{n[6:]} {100*v/tot:.1f}" for v, n in top) + f"   | {g['first']}")
