#!/bin/bash
# Config-5 evidence at full size on one B200: the run() timeline (PS_TIMELINE),
# the launch list, and ncu --set full captures of the two int8 GEMMs.
# usage (on the GPU box): bash tools/prof_config5.sh <tag>
set -u
OUT=gpurun_out/c5_${1:-x}
mkdir -p $OUT
PS_TIMELINE=1 REPS=2 timeout 600 python tools/e2e_trace.py 5 > $OUT/timeline.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $OUT/launches_5.csv \
  python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline --no-legs --e2e-steps 0 > /dev/null 2>&1
python tools/summarize_launches.py $OUT/launches_5.csv $OUT/launches_5.json > $OUT/launches_5.txt 2>/dev/null
for k in cross_gemm moment_gemm; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 2 -c 1 \
    -o $OUT/ncu_5_$k python tools/profile_one.py --config 5 > $OUT/ncu_5_$k.log 2>&1
done
echo done
