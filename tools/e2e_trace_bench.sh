for i in 1 2 3 4; do
  PS_TRACE=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /tmp/o.txt 2> /tmp/e.txt
  python -c "import json; d=json.loads(open('/tmp/o.txt').read().strip().splitlines()[-1]); print('E2E', round(d['e2e']['ms_per_step'],2))"
  grep "ps_run" /tmp/e.txt | tail -30 | awk '{k=$2; v=$(NF-1); s[k]=s[k]" "v} END {for (k in s) print k, s[k]}'
done
