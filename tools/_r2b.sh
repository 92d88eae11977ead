mkdir -p gpurun_out/r2b
timeout 600 python -m pytest tests/test_gpu_distributed.py -q -x > gpurun_out/r2b/dist.txt 2>&1
echo "rc=$?" >> gpurun_out/r2b/dist.txt
for w in vascular hub64; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:native_ensemble_kernel -c 1 \
    -o gpurun_out/r2b/ncu_$w python bench.py --workload $w --steps 1 --warmup 0 --no-extras --no-cpu \
    > gpurun_out/r2b/ncu_$w.log 2>&1
  echo "$w rc=$?"
done
echo done
