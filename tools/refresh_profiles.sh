#!/bin/bash
# Re-measure every BASELINE config on one B200 and refresh profiles/:
#   the default bench line (config 5 + legs + CPU baseline + e2e), one bench
#   line per config, ncu launch lists (time + DRAM bytes per launch) and
#   ncu --set full reports of the dominant kernels.
# usage (on the GPU box): bash tools/refresh_profiles.sh <round tag, e.g. r02> [full]
set -u
TAG=${1:-r02}
OUT=gpurun_out/prof_$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
timeout 1200 python bench.py > $OUT/bench_default.jsonl 2> $OUT/bench_default.err
tail -1 $OUT/bench_default.jsonl | cut -c1-300
CFGS=("1" "2" "3" "4 --test anova" "4 --test ttest" "4 --test kruskal" "4 --test mwu" "5s")
for c in "${CFGS[@]}"; do
  n=$(echo $c | sed 's/ --test /_/')
  extra="--no-cpu-baseline --no-legs"
  case "$n" in 2|3|4_anova|4_kruskal) extra="--no-legs" ;; esac
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 $extra > $OUT/bench_$n.jsonl 2> $OUT/bench_$n.err
  tail -1 $OUT/bench_$n.jsonl | cut -c1-200
done
# launch lists (cold-cache, serialised: shares, not absolutes)
CFGL=("5" "1" "2" "3" "4 --test anova" "4 --test ttest" "4 --test kruskal" "4 --test mwu" "5s")
for c in "${CFGL[@]}"; do
  n=$(echo $c | sed 's/ --test /_/')
  w=3; [ "$n" = "5" ] && w=1
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $OUT/launches_$n.csv \
    python bench.py --config $c --steps 1 --warmup $w --no-cpu-baseline --no-legs --e2e-steps 0 > /dev/null 2>&1
  python tools/summarize_launches.py $OUT/launches_$n.csv $OUT/launches_$n.json > $OUT/launches_$n.txt 2>/dev/null
done
if [ "${2:-}" = "full" ]; then
  # the int8 GEMMs at half scale (F = 10000: full 74-cluster waves), one mid-run launch each
  for spec in "cross_gemm:12" "moment_gemm:6"; do
    k=${spec%%:*}; skip=${spec##*:}
    timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s $skip -c 1 \
      -o $OUT/ncu_5_s0.5_$k python tools/profile_one.py --config 5 --scale 0.5 > $OUT/ncu_5_$k.log 2>&1
  done
  for spec in "2:spearman_walk" "5s:spearman_walk" "3:onehot_gemm_mc" "4 --test kruskal:rank_mixed_walk" "4 --test anova:group_gemm"; do
    c=${spec%%:*}; k=${spec##*:}
    n=$(echo $c | sed 's/ --test /_/; s/ --scale /_s/')
    timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 \
      -o $OUT/ncu_${n}_$k python tools/profile_one.py --config $c > $OUT/ncu_${n}.log 2>&1
  done
fi
echo done
