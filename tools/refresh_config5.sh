#!/bin/bash
# Re-measure only the config-5 artifacts of profiles/<tag>: default bench line, launch list, GEMM captures.
set -u
TAG=${1:-r02}
OUT=gpurun_out/prof5_$TAG
mkdir -p $OUT
timeout 1200 python bench.py > $OUT/bench_default.jsonl 2> $OUT/bench_default.err
tail -1 $OUT/bench_default.jsonl | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $OUT/launches_5.csv \
  python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline --no-legs --e2e-steps 0 > /dev/null 2>&1
python tools/summarize_launches.py $OUT/launches_5.csv $OUT/launches_5.json > $OUT/launches_5.txt 2>/dev/null
for spec in "cross_gemm:12" "moment_gemm:6"; do
  k=${spec%%:*}; skip=${spec##*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s $skip -c 1 \
    -o $OUT/ncu_5_s0.5_$k python tools/profile_one.py --config 5 --scale 0.5 > $OUT/ncu_5_$k.log 2>&1
done
echo done
