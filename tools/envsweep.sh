# Sweep one environment knob over bench workloads: VAR=GSDE_SLOTS VALS="1 2" WORKLOADS="hub64" bash tools/envsweep.sh
for w in ${WORKLOADS:-star3 hub64 vascular}; do for v in ${VALS}; do
  env $VAR=$v timeout 300 python bench.py --workload $w --no-cpu --no-extras --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$w','$VAR=$v', '%.4g'%d['value'], 'frac=%.3f'%d['roofline']['frac'], 'c=%.4f'%d['crossings_per_pstep'], d['step_ms'])"
done; done
