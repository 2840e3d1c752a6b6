#!/bin/bash
# Interleaved bench of several in-tree builds (libsprout_<V>.so) on one box.
# Usage: bash tools/gpu_abn.sh TAG "V1 V2 ..." CONFIG [CONFIG...]
TAG=$1; VARS=$2; shift 2
mkdir -p gpurun_out
for C in "$@"; do
  for rep in 1 2; do
    for V in $VARS; do
      export SPROUT_LIB_NAME=libsprout_$V.so
      timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abn_${TAG}_${C}_${V}${rep}.json 2>/dev/null
      python -c "import json; d=json.load(open('gpurun_out/abn_${TAG}_${C}_${V}${rep}.json')); print('$C $V$rep', 'value %.4g'%d['value'], 'ms %.3f'%d['ms_per_step'], 'sim_ms %.3f'%d['roofline']['launch_ms'])"
    done
  done
done
