mkdir -p gpurun_out/sweep
for c in 1 2 3 "4 --test anova" "4 --test ttest" "4 --test kruskal" "4 --test mwu" 5 5s; do
  n=$(echo $c | tr -d ' -')
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/sweep/$n.json 2> gpurun_out/sweep/$n.err
  python - gpurun_out/sweep/$n.json <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
  r=d.get("roofline",{})
  print(d["config"].get("config"), d["config"].get("test"), "ms=%.3f"%d["ms_per_step"], "e2e=%.3g"%d["e2e"]["value"], "kern=%s frac=%.3f ach=%.4g"%(r.get("kernel"), r.get("frac",0), r.get("achieved",0)), d.get("gpu_launches"))
except Exception as e: print(sys.argv[1], "ERR", e)
PY
done
