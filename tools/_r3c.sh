mkdir -p gpurun_out/r3c
timeout 600 python tools/e2e_star3_probe.py > gpurun_out/r3c/probe.txt 2>&1
echo done
