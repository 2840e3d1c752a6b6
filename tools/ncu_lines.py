#!/usr/bin/env python3
"""Per-CUDA-source-line instruction and stall-sample totals of an ncu report
(--import-source on, -lineinfo).  Usage: ncu_lines.py REP [TOP]"""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
samp = collections.Counter(); inst = collections.Counter(); text = {}
fname = "?"; cur = None; ix = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        ix = {k: i for i, k in enumerate(r)}; continue
    if ix is None or len(r) < 8:
        continue
    if r[0]:
        cur = (fname, int(r[0])); text[cur] = r[1].strip()[:90]; continue
    try:
        s = int(r[4] or 0); n = int(r[7] or 0)
    except ValueError:
        continue
    samp[cur] += s; inst[cur] += n
ts = sum(samp.values()); ti = sum(inst.values())
print(f"total samples {ts}  warp instructions {ti}")
for k, s in samp.most_common(top):
    print(f"{100*s/ts:5.1f}%  {100*inst[k]/ti:5.1f}%i  {k[0]}:{k[1]:<5d} {text.get(k,'')}")
