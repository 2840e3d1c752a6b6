#!/usr/bin/env python3
"""Executed warp instructions per SASS opcode of an ncu report.  Usage: ncu_opmix.py REP"""
import collections, csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]; ix = {k: i for i, k in enumerate(h)}
op = collections.Counter()
for r in rows[2:]:
    try:
        n = int(r[ix["Instructions Executed"]] or 0)
    except (ValueError, IndexError):
        continue
    src = r[ix["Source"]].strip()
    if src.startswith("@"):
        src = src.split(None, 1)[1]
    op[src.split()[0]] += n
tot = sum(op.values())
print("total", tot)
for k, v in op.most_common(40):
    print(f"{k:24s} {v:14d} {100*v/tot:5.1f}%")
