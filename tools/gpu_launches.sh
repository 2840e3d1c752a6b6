#!/bin/bash
# Per-kernel durations (ncu launch list, cold-cache serialised) of one bench step per variant.
# Usage: bash tools/gpu_launches.sh TAG "V1 V2 ..." CONFIG [extra bench args]
TAG=$1; VARS=$2; C=$3; shift 3
mkdir -p gpurun_out
for V in $VARS; do
  export SPROUT_LIB_NAME=libsprout_$V.so
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_${TAG}_${C}_${V}.csv python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline --no-e2e "$@" > /dev/null 2>&1
  python - "$V" gpurun_out/launch_${TAG}_${C}_${V}.csv << 'PY'
import csv, sys, collections
V, path = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value"); ui = hdr.index("Metric Unit")
tot = collections.OrderedDict(); cnt = collections.Counter()
for r in rows[1:]:
    name = r[ki].split("(")[0][:40]; v = float(r[vi].replace(",", "")); u = r[ui]
    v = v / 1e3 if u == "nsecond" else (v if u == "usecond" else v * 1e3)
    tot[name] = tot.get(name, 0) + v; cnt[name] += 1
print(V, " | ".join(f"{k} x{cnt[k]} {tot[k]/cnt[k]:.1f}us" for k in tot if "sprout" in k or "kernel" in k))
PY
done
