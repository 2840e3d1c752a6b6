#!/bin/bash
# functional test of bench.py's N > 1 path on a one-GPU box (ranks share the GPU over gloo; timings meaningless)
export SPROUT_BENCH_SHARE_GPU=1
P=29511
for args in "" "--config C2 --closed-loop 200" "--config C2 --scheme static" "--config C3"; do
  P=$((P+1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e $args > gpurun_out/share2.json 2> gpurun_out/share2.err
  echo "[$args] rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/share2.json'))
print(d['n_gpus'], d['value'], d['roofline']['frac'], d['check'], d.get('cpu_baseline'))" 2>&1 | tail -2; tail -2 gpurun_out/share2.err
done
