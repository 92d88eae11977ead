# A/B: alternate two library builds over the bench workloads, R rounds.
# usage: A=path/to/libgsde.so B=path/to/libgsde.so WORKLOADS="star3" R=2 bash tools/ab.sh
for r in $(seq ${R:-2}); do for w in ${WORKLOADS:-star3 hub64 vascular}; do for v in A B; do
  lib=${!v}
  GSDE_LIB_PATH=$lib timeout 300 python bench.py --workload $w --no-cpu --no-extras --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v','$w', '%.4g'%d['value'], 'frac=%.3f'%d['roofline']['frac'], d['clocks'], d['step_ms'])"
done; done; done
