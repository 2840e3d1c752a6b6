#!/bin/bash
TAG=${1:-cl}
mkdir -p gpurun_out
timeout 600 python bench.py --config C4 --closed-loop 1000 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_cl_$TAG.json 2> gpurun_out/bench_cl_$TAG.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/bench_cl_$TAG.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cl_window -c 1 -o gpurun_out/prof_cl_$TAG python bench.py --config C4 --closed-loop 1000 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_cl_$TAG.log 2>&1; echo "ncu rc=$?"
