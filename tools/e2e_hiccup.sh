# per-step e2e times of bench.py under a few settings (hiccup hunt)
run() { PS_BENCH_VERBOSE=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 8 $2 > /tmp/o.txt 2> /tmp/e.txt; echo "$1: $(grep 'e2e step' /tmp/e.txt | awk '{printf "%.1f ", $4}')"; }
for c in "${@:-2}"; do
  for i in 1 2; do run "$c" "--config $c"; done
done
