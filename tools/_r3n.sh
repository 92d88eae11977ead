mkdir -p gpurun_out/r3n
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r3n/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r3n/pytest_gpu.txt
echo done
