mkdir -p gpurun_out/r2n
timeout 900 python tools/e2e_probe.py > gpurun_out/r2n/probe.txt 2>&1
nvidia-smi -q | grep -i -A3 "PCIe Generation\|Link Width" >> gpurun_out/r2n/probe.txt
echo done
