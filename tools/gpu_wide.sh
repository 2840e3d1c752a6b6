#!/bin/bash
# wide-kernel bring-up: parity tests on the default build, then interleaved C4 timing of variants
mkdir -p gpurun_out
TAG=${1:-wide}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "wide or c4 or c2 or levels_classes or empty or large_tokens or full_size" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_$TAG.log
bash tools/gpu_exp.sh $TAG "new old ws7" C4 2
