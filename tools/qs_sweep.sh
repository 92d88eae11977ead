# Sweep (trips per iteration, vertex slots) pairs: PAIRS="10:1 14:2" WORKLOADS="hub64" bash tools/qs_sweep.sh
for w in ${WORKLOADS:-star3 hub64 vascular}; do for pq in ${PAIRS}; do
  q=${pq%:*}; sl=${pq#*:}
  GSDE_RARE_Q=$q GSDE_SLOTS=$sl timeout 300 python bench.py --workload $w --no-cpu --no-extras --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$w','Q=$q','slots=$sl', '%.4g'%d['value'], 'frac=%.3f'%d['roofline']['frac'], 'ms=%.2f'%min(d['step_ms']))"
done; done
