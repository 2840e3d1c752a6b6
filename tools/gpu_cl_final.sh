#!/bin/bash
# Re-measure the closed-loop lines and its ncu capture after a closed-loop
# change, plus the full GPU test suite.  Usage: bash tools/gpu_cl_final.sh TAG
TAG=${1:-clf}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --config C2 --closed-loop 1000 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_C2_closed_loop_$TAG.json 2>/dev/null; echo "closed loop C2 rc=$?"
timeout 900 python bench.py --config C4 --closed-loop 1000 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_C4_closed_loop_$TAG.json 2>/dev/null; echo "closed loop C4 rc=$?"
timeout 900 python bench.py --config C4 --closed-loop 1000 --q-update --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_C4_closed_loop_q_$TAG.json 2>/dev/null; echo "closed loop q C4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cl_window -c 1 -o gpurun_out/prof_cl_$TAG python bench.py --config C4 --closed-loop 1000 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_cl_$TAG.log 2>&1; echo "ncu-cl rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cl_$TAG.csv python bench.py --config C4 --closed-loop 1000 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu-launch rc=$?"
R=prof_cl_$TAG
if [ -f gpurun_out/$R.ncu-rep ]; then
  python tools/ncu_summary.py gpurun_out/$R.ncu-rep > gpurun_out/${R}_summary.txt 2>&1
  python tools/ncu_lines.py gpurun_out/$R.ncu-rep 60 > gpurun_out/${R}_lines.txt 2>&1
  rm -f gpurun_out/$R.ncu-rep
fi
