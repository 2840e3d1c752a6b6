#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py; logs in gpurun_out/
mkdir -p gpurun_out
for T in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_$T.log 2>&1
  echo "$T rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/sanitize_$T.log | tail -1)"
done
