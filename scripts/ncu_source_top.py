#!/usr/bin/env python
"""Top SASS lines of an ncu --page source --csv dump by stall samples."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
iS = h.index('Warp Stall Sampling (All Samples)')
iE = h.index('Instructions Executed')
tot = sum(int(r[iS]) for r in data)
toti = sum(int(r[iE]) for r in data)
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.006
print('samples', tot, 'warp-instructions', toti)
for r in data:
    if int(r[iS]) > tot * frac or int(r[iE]) > toti * frac * 2:
        print(r[0][-5:], r[1][:64].ljust(64), r[iS].rjust(6), r[iE].rjust(10))
