mkdir -p gpurun_out/r3m
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r3m/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r3m/pytest_gpu.txt
timeout 300 python tools/bigrun_time.py > gpurun_out/r3m/big.txt 2>&1
GSDE_CHUNK_PARTICLES=1000000000000 timeout 600 python tools/bigrun_time.py >> gpurun_out/r3m/big.txt 2>&1
echo done
