#!/bin/bash
# ncu --set full capture of the trace kernel for variant builds.  Usage: bash tools/gpu_prof.sh TAG "V1 V2" CONFIG
TAG=$1; VARS=$2; C=$3; shift 3
mkdir -p gpurun_out
for V in $VARS; do
  export SPROUT_LIB_NAME=libsprout_$V.so
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"trace_(wide_)?kernel" -s 2 -c 1 -o gpurun_out/prof_${TAG}_$V python bench.py --config $C --steps 2 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/ncu_${TAG}_$V.log 2>&1; echo "$V ncu rc=$?"
done
