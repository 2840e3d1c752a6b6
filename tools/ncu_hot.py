#!/usr/bin/env python3
"""Per-SASS-instruction stall attribution of an ncu report (source page).
Prints the instructions of the hottest executed region in address order with
their stall samples split by reason.  Usage: ncu_hot.py REP [min_exec] [max_lines]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
min_exec = int(sys.argv[2]) if len(sys.argv) > 2 else 1000000
maxl = int(sys.argv[3]) if len(sys.argv) > 3 else 300
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]; ix = {k: i for i, k in enumerate(h)}
reasons = ["stall_wait", "stall_dispatch", "stall_long_sb", "stall_short_sb", "stall_math", "stall_no_inst",
           "stall_not_selected", "stall_selected", "stall_branch_resolving", "stall_mio", "stall_lg"]
tot = {r: 0 for r in reasons}; allsum = 0; out = []
for r in rows[2:]:
    try:
        n = int(r[ix["Instructions Executed"]] or 0)
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, IndexError):
        continue
    allsum += s
    if n < min_exec:
        continue
    vals = {k: int(r[ix[k]] or 0) for k in reasons}
    for k in reasons: tot[k] += vals[k]
    out.append((r[ix["Address"]][-5:], n, s, vals, r[ix["Source"]].strip()))
print("samples in region", sum(x[2] for x in out), "of", allsum)
print("by reason:", {k.replace("stall_", ""): v for k, v in sorted(tot.items(), key=lambda x: -x[1])})
for a, n, s, v, t in out[:maxl]:
    top = sorted(((v[k], k.replace("stall_", "")) for k in reasons if v[k]), reverse=True)[:3]
    print(f"{a} {n:9d} {s:5d}  {' '.join(f'{k}:{c}' for c, k in top):40s} {t[:70]}")
