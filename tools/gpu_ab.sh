#!/bin/bash
# A/B bench of libsprout_A.so vs libsprout.so on the same box, interleaved.
# Usage: bash tools/gpu_ab.sh TAG CONFIG [CONFIG...]
TAG=$1; shift
mkdir -p gpurun_out
for C in "$@"; do
  for rep in 1 2; do
    for V in A B; do
      if [ $V = A ]; then export SPROUT_LIB_NAME=libsprout_A.so; else export SPROUT_LIB_NAME=libsprout.so; fi
      timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${TAG}_${C}_${V}${rep}.json 2>/dev/null
      python -c "import json; d=json.load(open('gpurun_out/ab_${TAG}_${C}_${V}${rep}.json')); print('$C $V$rep', 'value %.4g'%d['value'], 'ms %.3f'%d['ms_per_step'], 'sim_ms %.3f'%d['roofline']['launch_ms'])"
    done
  done
done
