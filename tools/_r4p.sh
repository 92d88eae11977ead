mkdir -p gpurun_out/r4p
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ref_ensemble_kernel -c 1 \
  -o /tmp/ncu_ref python bench.py --workload star3_ref --steps 1 --warmup 0 --no-extras --no-cpu > gpurun_out/r4p/ncu.log 2>&1
python tools/ncu_summary.py /tmp/ncu_ref.ncu-rep > gpurun_out/r4p/sum.json 2>&1
python tools/ncu_lines.py /tmp/ncu_ref.ncu-rep 50 > gpurun_out/r4p/lines.txt 2>&1
echo done
