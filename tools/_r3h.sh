mkdir -p gpurun_out/r3h
timeout 1500 python tools/trials_scale_check.py gpurun_out/r3h/trials_scale.csv > gpurun_out/r3h/trials.txt 2>&1
echo done
