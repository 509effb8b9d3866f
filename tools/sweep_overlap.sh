# e2e (ps_run from numpy) of config 2 Spearman: staging chunk x walk item size
export REPS=9
for C in ${CHUNKS:-16 8}; do for G in ${GBS:-16 32 64}; do
  r=$(PS_STAGE_CHUNK_MB=$C PS_SPEARMAN_GB=$G python tools/e2e_trace.py 2 spearman 2>&1 | grep summary)
  echo "chunk $C gb $G: $r"
  r=$(PS_STAGE_FLAT=1 PS_STAGE_CHUNK_MB=$C PS_SPEARMAN_GB=$G python tools/e2e_trace.py 2 spearman 2>&1 | grep summary)
  echo "chunk $C gb $G flat: $r"
done; done
r=$(PS_NO_OVERLAP=1 python tools/e2e_trace.py 2 spearman 2>&1 | grep summary); echo "no overlap: $r"
