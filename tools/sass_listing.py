#!/usr/bin/env python
"""Address-ordered SASS listing of the first kernel instance in an ncu source-page CSV
(`ncu -i rep --page source --csv --print-source sass`), instructions executed above a floor.
    python tools/sass_listing.py sass.csv [min_executions]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
floor = float(sys.argv[2]) if len(sys.argv) > 2 else 1e7
hdr = rows[1]
iex, isrc, ith = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Thread Instructions Executed")
ismp = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr) and r[0] != "Address":
        data.append(r)
tot = sum(int(r[iex] or 0) for r in data)
ts = sum(int(r[ismp] or 0) for r in data)
print("total warp-instructions %d, stall samples %d" % (tot, ts))
for i, r in enumerate(data):
    ex = int(r[iex] or 0)
    if ex > floor:
        print("%4d %7.1fM act %4.1f smp %5.2f%% %s" % (i, ex / 1e6, int(r[ith]) / ex, 100 * int(r[ismp] or 0) / ts,
                                                   r[isrc].strip()))
