#!/bin/bash
# Interleaved timing of in-tree variant builds (libsprout_<V>.so) on one box:
# bench.py's simulate (prep + trace) CUDA-event time per variant.
# Usage: bash tools/gpu_exp.sh TAG "V1 V2 ..." CONFIG [REPS] [extra bench args]
TAG=$1; VARS=$2; C=$3; REPS=${4:-2}; shift 4
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
for rep in $(seq 1 $REPS); do
  for V in $VARS; do
    export SPROUT_LIB_NAME=libsprout_$V.so
    timeout 300 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline --no-e2e "$@" > gpurun_out/exp_${TAG}_${C}_${V}${rep}.json 2> gpurun_out/exp_${TAG}_${C}_${V}${rep}.err
    python -c "import json; d=json.load(open('gpurun_out/exp_${TAG}_${C}_${V}${rep}.json')); print('$C %-10s'%'$V$rep', 'ms %.3f'%d['ms_per_step'], 'sim_ms %.4f'%d['roofline']['launch_ms'], 'frac %.3f'%d['roofline']['frac'], 'clk', d.get('clocks',{}).get('sm_mhz'))" 2>/dev/null || tail -3 gpurun_out/exp_${TAG}_${C}_${V}${rep}.err
  done
done
