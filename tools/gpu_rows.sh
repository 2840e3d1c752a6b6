#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trace_x1g -s 3 -c 1 -o gpurun_out/prof_x1g python bench.py --config C3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-fp64-check > /dev/null 2>&1; echo "x1g rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trace_x1_kernel -s 2 -c 1 -o gpurun_out/prof_x1 python bench.py --config C5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-fp64-check > /dev/null 2>&1; echo "x1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oracle_scheme -c 1 -o gpurun_out/prof_orc2 python bench.py --config C4 --scheme oracle --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "orc rc=$?"
for R in prof_x1g prof_x1 prof_orc2; do
  python tools/ncu_summary.py gpurun_out/$R.ncu-rep > gpurun_out/${R}_summary.txt 2>&1
  python tools/ncu_lines.py gpurun_out/$R.ncu-rep 40 > gpurun_out/${R}_lines.txt 2>&1
  rm -f gpurun_out/$R.ncu-rep
done
