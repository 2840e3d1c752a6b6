#!/bin/bash
# build variant V with extra nvcc flags into libsprout_V.so
V=$1; shift
cd /root/repo
rm -rf /tmp/bv_$V; mkdir -p /tmp/bv_$V
cp -r paper_2403_12900_b200 include /tmp/bv_$V/
rm -f /tmp/bv_$V/paper_2403_12900_b200/libsprout*.so
(cd /tmp/bv_$V && SPROUT_NVCC_EXTRA="$*" python -m paper_2403_12900_b200.build --force > /dev/null) || exit 1
cp /tmp/bv_$V/paper_2403_12900_b200/libsprout.so paper_2403_12900_b200/libsprout_$V.so
cuobjdump -res-usage paper_2403_12900_b200/libsprout_$V.so 2>/dev/null | grep -A1 "trace_kernelILi3ELb0" | tail -1 | sed "s/^/$V: /"
