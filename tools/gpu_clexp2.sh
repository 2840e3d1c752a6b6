#!/bin/bash
# Closed-loop A/B on one box: the chain-count (wave) sweep of tools/cl_tail.py
# and interleaved C4 --closed-loop 1000 runs of variant builds.
# Usage: bash tools/gpu_clexp2.sh TAG "V1 V2 ..." [X ...]
TAG=$1; VARS=$2; shift 2
mkdir -p gpurun_out
for V in $VARS; do
  SPROUT_LIB_NAME=libsprout_$V.so timeout 600 python tools/cl_tail.py "$@" > gpurun_out/cltail_${TAG}_$V.txt 2>&1; echo "tail $V rc=$?"; sed "s/^/$V /" gpurun_out/cltail_${TAG}_$V.txt | tail -8
done
for rep in 1 2; do
  for V in $VARS; do
    SPROUT_LIB_NAME=libsprout_$V.so timeout 600 python bench.py --config C4 --closed-loop 1000 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/clexp_${TAG}_${V}$rep.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/clexp_${TAG}_${V}$rep.json')); print('$V$rep', 'ms %.2f' % d['ms_per_step'])" 2>/dev/null || echo "$V$rep failed"
  done
done
