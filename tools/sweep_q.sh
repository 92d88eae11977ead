# Sweep the ensemble kernel's trips-per-iteration (GSDE_RARE_Q) over the bench workloads.
for w in ${WORKLOADS:-star3 hub64 vascular}; do for q in ${QS:-4 6 8 12}; do
  GSDE_RARE_Q=$q timeout 300 python bench.py --workload $w --no-cpu --no-extras --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$w','q=$q', '%.4g'%d['value'], 'frac=%.3f'%d['roofline']['frac'], 'c=%.4f'%d['crossings_per_pstep'])"
done; done
