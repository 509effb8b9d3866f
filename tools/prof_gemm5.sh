#!/bin/bash
# Sustained tcgen05 i8 peak + ncu --set full captures of the config-5 int8 GEMMs
# (cross_gemm_mc, moment_gemm_mc) at half scale (F = 10000: full 74-cluster waves).
# usage (GPU box): bash tools/prof_gemm5.sh <out dir under gpurun_out>
set -u
OUT=gpurun_out/${1:-gemm5}
mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tc05_peak tools/microbench/tc05_peak.cu -lcuda && /tmp/tc05_peak > $OUT/tc05_peak.json
cat $OUT/tc05_peak.json
SC=${2:-0.5}
for spec in "cross_gemm:12" "moment_gemm:6"; do
  k=${spec%%:*}; skip=${spec##*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s $skip -c 1 \
    -o $OUT/ncu_5_s${SC}_$k python tools/profile_one.py --config 5 --scale $SC > $OUT/ncu_$k.log 2>&1
  tail -2 $OUT/ncu_$k.log
done
echo done
