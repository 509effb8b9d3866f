j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['e2e']['ms_per_step'],2), round(d['ms_per_step'],2))"; }
echo "default: $(python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 6 2>/dev/null | j)"
echo "omp passive: $(OMP_WAIT_POLICY=PASSIVE python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 6 2>/dev/null | j)"
echo "blas1: $(OPENBLAS_NUM_THREADS=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 6 2>/dev/null | j)"
echo "default again: $(python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 6 2>/dev/null | j)"
REPS=9 python tools/e2e_trace.py 2 spearman 2>&1 | grep summary
nproc; python -c "import torch; print(torch.get_num_threads())"
