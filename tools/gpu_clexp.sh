for rep in 1 2; do for V in base b3; do
  export SPROUT_LIB_NAME=libsprout_$V.so
  timeout 300 python bench.py --config C4 --closed-loop 1000 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$V', round(d['ms_per_step'],2))"
done; done
export SPROUT_LIB_NAME=libsprout_base.so
timeout 900 python -m pytest tests/test_gpu_closed_loop.py -q -x 2>&1 | tail -2
