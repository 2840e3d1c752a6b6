#!/usr/bin/env python3
"""Per-CUDA-source-line stall samples and instruction counts from an ncu
report (needs -lineinfo).  Usage: ncu_lines.py REP [TOP]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = {}
fname = ""; line = None; src = ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if len(r) < 8 or r[0] == "Line No":
        continue
    if r[0] != "":
        line = (fname, r[0]); src = r[1]; continue
    try:
        s = int(r[4] or 0); n = int(r[7] or 0)
    except ValueError:
        continue
    a = agg.setdefault(line, [0, 0, src])
    a[0] += s; a[1] += n
tot = sum(v[0] for v in agg.values()) or 1
for (f, l), (s, n, src) in sorted(agg.items(), key=lambda t: -t[1][0])[:top]:
    print(f"{100*s/tot:5.1f}% {n:12d} {f}:{l:5s} {src.strip()[:80]}")
