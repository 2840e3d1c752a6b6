#!/bin/bash
# Full round measurement on one B200: build, GPU parity tests, smoke, the
# default bench line (C4, with cpu_baseline + e2e), the reference arm, extra
# config / scheme / NEXT lines, the ncu launch list of the default bench and
# ncu --set full captures of the trace kernel, the other kernels and the
# closed-loop chain kernel.   Usage: bash tools/gpu_full.sh TAG
TAG=${1:-full}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/nvsmi_$TAG.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"; cut -c1-300 gpurun_out/bench_ref_$TAG.json
timeout 600 python bench.py --graph --no-e2e --no-cpu-baseline > gpurun_out/bench_C4_graph_$TAG.json 2> gpurun_out/bench_C4_graph_$TAG.err; echo "graph rc=$?"
for C in C2 C3 C5; do
  timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --cpu-seconds 8 > gpurun_out/bench_${C}_$TAG.json 2> gpurun_out/bench_${C}_$TAG.err; echo "bench $C rc=$?"; cut -c1-300 gpurun_out/bench_${C}_$TAG.json
done
for SC in co2opt static oracle; do
  timeout 900 python bench.py --config C4 --scheme $SC --steps 10 --warmup 3 --no-e2e --cpu-seconds 8 > gpurun_out/bench_C4_${SC}_$TAG.json 2> gpurun_out/bench_C4_${SC}_$TAG.err; echo "bench C4 $SC rc=$?"; cut -c1-300 gpurun_out/bench_C4_${SC}_$TAG.json
done
timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --preference --request-cdf 32 > gpurun_out/bench_C4_next4_$TAG.json 2> gpurun_out/bench_C4_next4_$TAG.err; echo "next4 rc=$?"
timeout 600 python bench.py --config C2 --closed-loop 1000 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_C2_closed_loop_$TAG.json 2>/dev/null; echo "closed loop C2 rc=$?"
timeout 900 python bench.py --config C4 --closed-loop 1000 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_C4_closed_loop_$TAG.json 2>/dev/null; echo "closed loop C4 rc=$?"
timeout 900 python bench.py --config C4 --closed-loop 1000 --q-update --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_C4_closed_loop_q_$TAG.json 2>/dev/null; echo "closed loop q C4 rc=$?"
timeout 300 python bench.py --evaluator --steps 10 > gpurun_out/bench_evaluator_C4_$TAG.json 2>/dev/null; echo "evaluator rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu-launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 2 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu-full rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:'lp_solve|prep_kernel|reduce_stage' -s 6 -c 5 -o gpurun_out/prof_other_$TAG python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_other_$TAG.log 2>&1; echo "ncu-other rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cl_window -c 1 -o gpurun_out/prof_cl_$TAG python bench.py --config C4 --closed-loop 1000 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_cl_$TAG.log 2>&1; echo "ncu-cl rc=$?"
# summaries on the box (the .ncu-rep files are large; gpurun_out must stay < 64 MiB)
for R in prof_$TAG prof_other_$TAG prof_cl_$TAG; do
  [ -f gpurun_out/$R.ncu-rep ] || continue
  python tools/ncu_summary.py gpurun_out/$R.ncu-rep > gpurun_out/${R}_summary.txt 2>&1
  python tools/ncu_lines.py gpurun_out/$R.ncu-rep 60 > gpurun_out/${R}_lines.txt 2>&1
  python tools/ncu_opmix.py gpurun_out/$R.ncu-rep > gpurun_out/${R}_opmix.txt 2>&1
done
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/prof_${TAG}_traffic.csv 2>&1
rm -f gpurun_out/prof_other_$TAG.ncu-rep gpurun_out/prof_cl_$TAG.ncu-rep
du -sh gpurun_out
