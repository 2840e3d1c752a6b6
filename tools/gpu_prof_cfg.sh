#!/bin/bash
# ncu --set full capture of the trace kernel on one config.  Usage: bash tools/gpu_prof_cfg.sh TAG CONFIG
TAG=$1; CFG=$2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
timeout 600 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; cut -c1-200 gpurun_out/bench_$TAG.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 2 -c 1 -o gpurun_out/prof_$TAG python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu-full rc=$?"
