#!/usr/bin/env python
"""Print a kernel's SASS with per-instruction executed counts and stall samples from an
`ncu --page source --csv --print-source sass` export (read here, no GPU).
    python tools/sass_hot.py /tmp/sass.csv [min_exec_fraction]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
hdr = rows[1]
ia, isrc, ismp, iex, ith = (hdr.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                                    "Instructions Executed", "Thread Instructions Executed"))
data = []
for r in rows[2:]:
    if len(r) < len(hdr) or r[0] == "Address":
        if data:
            break  # first kernel instance only
        continue
    data.append(r)
tot_ex = sum(int(r[iex] or 0) for r in data)
tot_s = sum(int(r[ismp] or 0) for r in data)
print("total warp-instr %d, samples %d" % (tot_ex, tot_s))
for r in data:
    ex = int(r[iex] or 0)
    if ex < thr * tot_ex:
        continue
    th = int(r[ith] or 0)
    print("%5.2f%% ex  %5.2f%% smp  act %4.1f  %s" % (100.0 * ex / max(tot_ex, 1), 100.0 * int(r[ismp] or 0) / max(tot_s, 1),
                                                   th / ex if ex else 0, r[isrc].strip()))
