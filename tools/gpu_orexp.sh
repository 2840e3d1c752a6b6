for rep in 1 2; do for V in g100 t256g200 t256g300; do
  export SPROUT_LIB_NAME=libsprout_$V.so
  timeout 300 python bench.py --config C4 --scheme oracle --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$V', round(d['ms_per_step'],2))"
done; done
