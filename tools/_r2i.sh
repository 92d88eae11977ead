mkdir -p gpurun_out/r2i
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2i/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r2i/pytest_gpu.txt
for w in vascular hub64 star5_trials; do
  k=native_ensemble_kernel; [ "$w" = star5_trials ] && k=native_trials_kernel
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 \
    -o /tmp/ncu_$w python bench.py --workload $w --steps 1 --warmup 0 --no-extras --no-cpu \
    > gpurun_out/r2i/ncu_$w.log 2>&1
  echo "$w rc=$?"
  python tools/ncu_summary.py /tmp/ncu_$w.ncu-rep > gpurun_out/r2i/sum_$w.json 2>&1
  python tools/ncu_lines.py /tmp/ncu_$w.ncu-rep 80 > gpurun_out/r2i/lines_$w.txt 2>&1
  ncu -i /tmp/ncu_$w.ncu-rep --page source --csv --print-source sass > gpurun_out/r2i/sass_$w.csv 2>/dev/null
done
echo done
