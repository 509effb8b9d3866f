#!/bin/bash
# Per-kernel launch times (cold, serialised) of one bench config:
#   bash tools/launch_times.sh <out.csv> <bench args...>
out=$1; shift
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $out python bench.py "$@" --no-cpu-baseline --no-legs --e2e-steps 0 > /dev/null 2>&1
python tools/summarize_launches.py $out ${out%.csv}.json
