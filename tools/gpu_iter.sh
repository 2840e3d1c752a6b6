#!/bin/bash
# One GPU iteration: build, GPU parity tests, a bench line, an ncu capture of
# the trace kernel.  Usage: bash tools/gpu_iter.sh TAG [bench args...]
TAG=${1:-iter}; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
cat gpurun_out/bench_$TAG.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'ms',d['ms_per_step'],'frac',d['roofline']['frac'],'sim_ms',d['roofline']['launch_ms'],'lp',d['lp_cells_per_s'])"
tail -3 gpurun_out/bench_$TAG.err
if [ -z "$NO_NCU" ]; then
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e "$@" > /dev/null 2>&1; echo "ncu-launch rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 2 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu-full rc=$?"
fi
