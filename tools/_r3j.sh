mkdir -p gpurun_out/r3j
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_state_parity.py tests/test_gpu_c4.py -m gpu -q -s > gpurun_out/r3j/parity_s.txt 2>&1
echo "rc=$?" >> gpurun_out/r3j/parity_s.txt
echo done
