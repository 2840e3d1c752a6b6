#!/bin/bash
TAG=${1:-w}
mkdir -p gpurun_out
bash tools/gpu_exp.sh $TAG "new ws7 old" C4 1
export SPROUT_LIB_NAME=libsprout_new.so
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"trace_(wide_)?kernel" -s 2 -c 1 -o gpurun_out/prof_${TAG}_new python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu rc=$?"
