#!/bin/bash
# FP64 DMMA / DFMA peak microbenchmark (tools/fp64_peak.cu) with the SM clock sampled by
# nvidia-smi during the run — the roofline denominator and its clock record.
set -e
cd "$(dirname "$0")"
[ -x ./fp64_peak ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,power.draw --format=csv,noheader -lms 50 > /tmp/fp64_clocks.csv &
SMI=$!
sleep 0.5
./fp64_peak
./fp64_peak
kill $SMI
echo "== SM clocks during the run (MHz, sampled every 50 ms): min / median / max, and event-reason masks seen"
awk -F', ' '{gsub(/ MHz/,"",$1); print $1}' /tmp/fp64_clocks.csv | sort -n | awk '{a[NR]=$1} END {print a[1], a[int((NR+1)/2)], a[NR]}'
awk -F', ' '{print $3}' /tmp/fp64_clocks.csv | sort | uniq -c
