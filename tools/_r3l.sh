mkdir -p gpurun_out/r3l
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r3l/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r3l/pytest_gpu.txt
echo done
