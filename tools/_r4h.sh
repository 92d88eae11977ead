mkdir -p gpurun_out/r4h
timeout 900 ncu --set full --import-source on --clock-control none -k regex:native_ensemble_kernel -s 1 -c 1 \
  -o /tmp/ncu_pp1 python tools/star3_pp_vs_lean.py > gpurun_out/r4h/ncu.log 2>&1
python tools/ncu_lines.py /tmp/ncu_pp1.ncu-rep 70 > gpurun_out/r4h/lines_pp.txt 2>&1
echo done
