#!/usr/bin/env python3
"""Summarise an ncu --set full report: key metrics WITH UNITS (raw page), all
stall reasons per issued instruction, and optionally (--sass) the hottest SASS
instructions by stall samples with their dominant reason.
Usage: ncu_summary.py REP [--kernel REGEX] [--sass [N]]"""
import collections, csv, io, re, subprocess, sys

rep = sys.argv[1]
kre = None
if "--kernel" in sys.argv:
    kre = re.compile(sys.argv[sys.argv.index("--kernel") + 1])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
unit = dict(zip(h, units))
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__block_size",
        "launch__grid_size", "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct"]
for r in rows[2:]:
    d = dict(zip(h, r))
    name = d.get("Kernel Name", "")
    if kre and not kre.search(name):
        continue
    print(name[:100])
    for k in keys:
        if k in d and d[k] != "":
            print(f"  {k:66s} {d[k]:>18s} {unit.get(k, '')}")
    st = {k: d[k] for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")}
    top = sorted(((float((v or "0").replace(",", "")), k) for k, v in st.items()), reverse=True)
    print("  stalls (warp-cycles per issued instruction):")
    for v, k in top:
        if v >= 0.01:
            print(f"    {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):28s} {v:.3f}")
if "--sass" in sys.argv:
    i = sys.argv.index("--sass")
    topn = int(sys.argv[i + 1]) if len(sys.argv) > i + 1 and sys.argv[i + 1].isdigit() else 40
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hi = next(j for j, r in enumerate(rows) if "Source" in r)
    h = rows[hi]
    ix = {k: j for j, k in enumerate(h)}
    items = []
    reasons = [k for k in h if k.startswith("stall_") or "Stall Sampling" in k]
    for r in rows[hi + 1:]:
        try:
            s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
            n = int(r[ix["Instructions Executed"]] or 0)
        except (ValueError, IndexError, KeyError):
            continue
        items.append((s, n, r[ix["Address"]] if "Address" in ix else "", r[ix["Source"]]))
    tot = sum(x[0] for x in items)
    print(f"samples {tot}")
    for s, n, a, src_ in sorted(items, reverse=True)[:topn]:
        print(f"  {100 * s / max(tot, 1):5.2f}%  exec {n:10d}  {a:>8s}  {src_[:90]}")
