#!/usr/bin/env python
"""Stall samples of an `ncu --page source --csv --print-source sass` export summed over SASS
index ranges (read here, no GPU).
    python tools/sass_regions.py sass.csv start1 start2 ...   (region k = [start_k, start_k+1))"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cuts = [int(x) for x in sys.argv[2:]]
hdr = rows[1]
iex = hdr.index("Instructions Executed")
cols = ["stall_long_sb", "stall_short_sb", "stall_wait", "stall_branch_resolving", "stall_math", "stall_mio",
        "stall_dispatch", "stall_no_inst", "stall_lg", "stall_selected", "stall_not_selected"]
ci = [hdr.index(c) for c in cols]
ni = hdr.index("Warp Stall Sampling (Not-issued Samples)")
data = []
for r in rows[2:]:
    if len(r) < len(hdr) or r[0] == "Address":
        if data:
            break
        continue
    data.append(r)
edges = [0] + cuts + [len(data)]
tot_ex = sum(int(r[iex] or 0) for r in data)
tot_n = sum(int(r[ni] or 0) for r in data)
print("region        ex%   notissued%  " + " ".join("%8s" % c.replace("stall_", "")[:8] for c in cols))
for a, b in zip(edges[:-1], edges[1:]):
    seg = data[a:b]
    ex = sum(int(r[iex] or 0) for r in seg)
    n = sum(int(r[ni] or 0) for r in seg)
    st = [sum(int(r[c] or 0) for r in seg) for c in ci]
    tot = max(1, sum(int(rr[c] or 0) for rr in data for c in ci))
    print("%4d-%4d  %6.2f  %8.2f    " % (a, b, 100.0 * ex / tot_ex, 100.0 * n / max(tot_n, 1)) +
          " ".join("%8.2f" % (100.0 * s / tot) for s in st))
