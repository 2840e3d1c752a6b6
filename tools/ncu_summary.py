#!/usr/bin/env python3
"""Summarise an ncu --set full report of the trace kernel: key metrics and
per-SASS-block instruction/stall hot spots.  Usage: ncu_summary.py REP [--sass]"""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__block_size",
        "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"]
for r in rows[2:]:
    d = dict(zip(h, r))
    print(d.get("Kernel Name", "")[:80])
    for k in keys:
        if k in d:
            print(f"  {k:70s} {d[k]}")
    st = {k: d[k] for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")}
    top = sorted(((float(v or 0), k) for k, v in st.items()), reverse=True)[:8]
    for v, k in top:
        print(f"  stall {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):30s} {v:.3f}")
if "--sass" in sys.argv:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    h = rows[1]
    ix = {k: i for i, k in enumerate(h)}
    byn = collections.Counter(); cnt = collections.Counter(); tot = 0; inst = 0
    for r in rows[2:]:
        try:
            n = int(r[ix["Instructions Executed"]] or 0); s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        except (ValueError, IndexError):
            continue
        byn[n] += s; cnt[n] += 1; tot += s; inst += n
    print("samples", tot, "warp instructions", inst)
    for n, s in byn.most_common(15):
        print(f"  exec {n:10d} x {cnt[n]:4d} instr: {s:7d} samples ({100 * s / tot:.1f}%)")
