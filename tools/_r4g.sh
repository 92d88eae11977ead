mkdir -p gpurun_out/r4g
timeout 900 ncu --set full --import-source on --clock-control none -k regex:native_ensemble_kernel -c 2 \
  -o /tmp/ncu_pp python tools/star3_pp_vs_lean.py > gpurun_out/r4g/ncu.log 2>&1
python tools/ncu_summary.py /tmp/ncu_pp.ncu-rep > gpurun_out/r4g/sum.json 2>&1
ncu -i /tmp/ncu_pp.ncu-rep --page raw --csv --metrics smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio > gpurun_out/r4g/raw.csv 2>&1
echo done
