#!/bin/bash
# A/B/A/B of the multicast vs CTA-pair int8 GEMMs on the config-5 bench line (same box).
for i in 1 2; do
  for m in 0 1; do
    PS_GEMM_2SM=$m timeout 600 python bench.py --no-cpu-baseline --no-legs --e2e-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('PS_GEMM_2SM=$m step %.1f ms frac %.3f clocks %s' % (d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz']))"
  done
done
