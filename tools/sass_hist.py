#!/usr/bin/env python
"""Executed-instruction histogram (per unit) of the profiled kernel in an ncu report.
usage: sass_hist.py REPORT.ncu-rep UNITS [TOP]"""
import csv, io, re, subprocess, sys
from collections import Counter

rep, units = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
iE = hdr.index("Instructions Executed")
C = Counter()
tot = 0
for r in data:
    n = int(r[iE] or 0)
    tot += n
    s = re.sub(r'^@!?U?P\w+\s+', '', r[1].strip())
    C[s.split()[0] if s else '?'] += n
print("warp instructions per unit: %.1f" % (tot / units))
for op, n in C.most_common(top):
    print("%-34s %7.2f" % (op, n / units))
