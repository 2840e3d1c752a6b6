#!/bin/bash
# build, GPU tests, bench lines for the listed configs (no ncu).  Usage: bash tools/gpu_quick.sh TAG C4 C3 ...
TAG=$1; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
for C in "$@"; do
  timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${C}_$TAG.json 2> gpurun_out/bench_${C}_$TAG.err
  python -c "import json,sys; d=json.load(open('gpurun_out/bench_${C}_$TAG.json')); print('$C', 'value %.4g'%d['value'], 'ms %.3f'%d['ms_per_step'], 'sim_ms %.3f'%d['roofline']['launch_ms'], 'frac %.3f'%d['roofline']['frac'])" || tail -5 gpurun_out/bench_${C}_$TAG.err
done
