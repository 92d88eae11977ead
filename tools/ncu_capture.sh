# Full ncu capture of the dominant native kernel for each bench workload (one GPU).
# usage: TAG=r01_v5 bash tools/ncu_capture.sh [workloads...]
TAG=${TAG:-cap}
for w in ${@:-star3 hub64 vascular star5_trials}; do
  k=native_ensemble_kernel; [ "$w" = star5_trials ] && k=native_trials_kernel
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 \
    -o gpurun_out/${TAG}_$w python bench.py --workload $w --steps 1 --warmup 0 --no-extras --no-cpu \
    > gpurun_out/${TAG}_$w.log 2>&1
  echo "$w ncu rc=$?"
done
