#!/bin/bash
TAG=${1:-cl}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_closed_loop.py -q -x > gpurun_out/pytest_cl_$TAG.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_cl_$TAG.log
timeout 600 python bench.py --config C4 --closed-loop 1000 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_cl_$TAG.json 2> gpurun_out/bench_cl_$TAG.err; echo "bench rc=$?"; cut -c1-250 gpurun_out/bench_cl_$TAG.json; tail -3 gpurun_out/bench_cl_$TAG.err
timeout 600 python bench.py --config C2 --closed-loop 1000 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_cl2_$TAG.json 2>&1; echo "bench C2 rc=$?"; cut -c1-250 gpurun_out/bench_cl2_$TAG.json
