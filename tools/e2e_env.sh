# bench e2e under a few host-side settings (noise check)
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['e2e']['ms_per_step'],2), round(d['ms_per_step'],2))"; }
for i in 1 2 3; do
echo "default: $(python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | j)"
echo "no prefault: $(PS_NO_PREFAULT=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | j)"
done
