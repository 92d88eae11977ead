mkdir -p gpurun_out/r3w
for w in vascular hub64; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:native_ensemble_kernel -c 1 \
    -o /tmp/ncu_$w python bench.py --workload $w --steps 1 --warmup 0 --no-extras --no-cpu > gpurun_out/r3w/ncu_$w.log 2>&1
  python tools/ncu_summary.py /tmp/ncu_$w.ncu-rep > gpurun_out/r3w/sum_$w.json 2>&1
  python tools/ncu_lines.py /tmp/ncu_$w.ncu-rep 60 > gpurun_out/r3w/lines_$w.txt 2>&1
done
echo done
