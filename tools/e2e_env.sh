# bench e2e under a few host-side settings (noise check)
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['e2e']['ms_per_step'],2), round(d['ms_per_step'],2))"; }
for i in 1 2 3 4; do
echo "default: $(python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | j)"
done
for i in 1 2 3 4; do
echo "bind: $(OMP_PROC_BIND=close OMP_PLACES=cores python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | j)"
done
for i in 1 2 3; do
echo "omp8: $(OMP_NUM_THREADS=8 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | j)"
done
python -c "
import torch, ctypes, sys
sys.path.insert(0,'.')
import paper_2505_00448_b200 as ps
from paper_2505_00448_b200 import _lib
_lib.load()
import os
maps=open('/proc/self/maps').read()
print(sorted({l.split()[-1] for l in maps.splitlines() if 'gomp' in l or 'omp' in l.split()[-1]}))
"
